# fused dH split-K slabs through TMA stores: parity, A/B
python paper_2605_21442_b200/build.py >/dev/null
timeout 1500 python -m pytest tests -m gpu -x -q -k "fused or kd or vocab_shard or token_parallel or nvls or single_rank" 2>&1 | tail -2
timeout 900 python scripts/sweep_env.py --config llama8b --path fused --reps 4 '' 'LCE_DH_SLAB_TMA=0'
timeout 900 python scripts/sweep_env.py --config llama1b --path fused --reps 4 '' 'LCE_DH_SLAB_TMA=0'
timeout 900 python scripts/sweep_env.py --config qwen7b --path fused --reps 4 '' 'LCE_DH_SLAB_TMA=0'
