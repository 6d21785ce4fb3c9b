python paper_2605_21442_b200/build.py >/dev/null
timeout 1200 python -m pytest tests -m gpu -x -q -k "tiny_config or ragged or random_shapes or fused_many or config_shapes_reduced or kd_matches or backward_adamw" 2>&1 | tail -2
bash scripts/ab_bench.sh paper_2605_21442_b200/liblce_base.so "llama8b llama1b" --no-split
bash scripts/ab_bench.sh paper_2605_21442_b200/liblce_base.so "llama8b" --no-split --path split
timeout 900 python scripts/sweep_env.py --config llama8b --path fused --reps 3 '' 'LCE_WIDE_2=1'
LCE_DBG_WAITS=1 python scripts/one_step.py --config llama8b --path fused --steps 1 2>&1 | grep "lce wide" | head -3
