python paper_2605_21442_b200/build.py >/dev/null
nproc; lscpu | grep -E "Model name|^CPU\(s\)"
timeout 600 python scripts/sweep_env.py --config llama8b --path fused --reps 3 '' 'LCE_DW_PREFETCH=0'
timeout 900 python scripts/sweep_env.py --config llama70b --path fused --reps 2 --steps 3 '' 'LCE_DW_PREFETCH=0'
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 2>&1 | tail -30
