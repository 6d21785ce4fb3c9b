# dW drain: TMA store / reduce-add (default) vs coalesced direct stores through a smem transpose
python paper_2605_21442_b200/build.py >/dev/null
LCE_DW_STORE=coalesced timeout 900 python -m pytest tests -m gpu -x -q -k "tiny_config or fused_many or random_shapes or fused_config_shapes or deterministic or grad_scale_sum" 2>&1 | tail -2
timeout 900 python scripts/sweep_env.py --config llama8b --path fused --reps 4 '' 'LCE_DW_STORE=coalesced'
timeout 900 python scripts/sweep_env.py --config llama8b --path split --reps 3 '' 'LCE_DW_STORE=coalesced'
timeout 900 python scripts/sweep_env.py --config llama1b --path fused --reps 4 '' 'LCE_DW_STORE=coalesced'
