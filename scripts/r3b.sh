# phased wide-tile schedule (LCE_WIDE_R): parity of the wide kernels, then A/B of R
python paper_2605_21442_b200/build.py >/dev/null
timeout 900 python -m pytest tests -m gpu -x -q -k "wide_schedules or debug_gemm or fused_many or random_shapes or tiny_config or fused_config_shapes" 2>&1 | tail -3
timeout 900 python scripts/sweep_env.py --config llama8b --path fused --reps 3 '' 'LCE_WIDE_R=0' 'LCE_WIDE_R=4' 'LCE_WIDE_R=12' 'LCE_WIDE_R=16'
timeout 600 python scripts/sweep_env.py --config llama8b --path split --reps 3 '' 'LCE_WIDE_R=0' 'LCE_WIDE_R=12'
timeout 600 python scripts/sweep_env.py --config llama1b --path fused --reps 3 '' 'LCE_WIDE_R=0' 'LCE_WIDE_R=12'
