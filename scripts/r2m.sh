python paper_2605_21442_b200/build.py >/dev/null
LCE_DW_STORE=mixed timeout 900 python -m pytest tests -m gpu -x -q -k "tiny_config or fused_many or random_shapes or grad_scale" 2>&1 | tail -2
timeout 600 python scripts/sweep_env.py --config llama8b --path fused --reps 4 '' 'LCE_DW_STORE=mixed'
timeout 600 python scripts/sweep_env.py --config llama8b --path split --reps 3 '' 'LCE_DW_STORE=mixed'
timeout 900 python scripts/sweep_env.py --config llama70b --path fused --reps 2 --steps 3 '' 'LCE_DW_STORE=mixed'
