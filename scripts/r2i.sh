python paper_2605_21442_b200/build.py >/dev/null
LCE_WIDE_SPLIT=1 timeout 900 python -m pytest tests -m gpu -x -q -k "random_shapes or tiny_config or ragged or fused_many or config_shapes_reduced" 2>&1 | tail -2
timeout 600 python scripts/sweep_env.py --config llama8b --path fused --reps 3 '' 'LCE_WIDE_SPLIT=1'
timeout 600 python scripts/sweep_env.py --config llama8b --path split --reps 3 '' 'LCE_WIDE_SPLIT=1'
timeout 600 python scripts/sweep_env.py --config llama1b --path fused --reps 3 '' 'LCE_WIDE_SPLIT=1'
timeout 900 python scripts/sweep_env.py --config llama70b --path fused --reps 2 --steps 3 '' 'LCE_WIDE_SPLIT=1'
timeout 600 python scripts/sweep_env.py --config qwen7b --path fused --reps 3 '' 'LCE_WIDE_SPLIT=1'
