set -x
nvidia-smi --query-gpu=name,clocks.sm,power.draw --format=csv
python paper_2605_21442_b200/build.py >/dev/null
timeout 900 python -m pytest tests -m gpu -x -q -k "tiny_config or ragged or random_shapes or grad_scale or vocab_shard_offsets or many_row_chunks or config_shapes_reduced" 2>&1 | tail -4
timeout 600 python scripts/sweep_env.py --config llama8b --path fused --reps 3 '' 'LCE_DW_STORE=tma'
timeout 600 python scripts/sweep_env.py --config llama8b --path split --reps 3 '' 'LCE_DW_STORE=tma'
timeout 600 python scripts/sweep_env.py --config llama1b --path fused --reps 3 '' 'LCE_DW_STORE=tma'
timeout 900 python scripts/sweep_env.py --config llama70b --path fused --reps 2 --steps 3 '' 'LCE_DW_STORE=tma'
