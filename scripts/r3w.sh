# new K-lockstep defaults (wide tiles + pair forward / G, 2 us poll): parity subset + A/B vs off and vs the previous default
python paper_2605_21442_b200/build.py >/dev/null
timeout 900 python -m pytest tests -m gpu -x -q -k "lockstep or wide_schedules or fused_deterministic or debug_gemm or tiny_config or random_shapes or graph" 2>&1 | tail -2
OLD="LCE_LOCK_2=0 LCE_LOCK_4=0"
timeout 900 python scripts/sweep_env.py --config llama8b --path fused --reps 4 'LCE_LOCK=0' "$OLD" ''
timeout 900 python scripts/sweep_env.py --config llama8b --path split --reps 3 'LCE_LOCK=0' "$OLD" ''
timeout 900 python scripts/sweep_env.py --config llama1b --path fused --reps 4 'LCE_LOCK=0' ''
timeout 900 python scripts/sweep_env.py --config llama1b --path split --reps 4 'LCE_LOCK=0' ''
timeout 900 python scripts/sweep_env.py --config qwen7b --path split --reps 3 'LCE_LOCK=0' ''
