# fused path with the forward's A rows gathered by TMA tile::gather4 (no H_c copy): parity, then A/B time and peak HBM
python paper_2605_21442_b200/build.py >/dev/null
timeout 1500 python -m pytest tests -m gpu -x -q -k "fused or autograd or vocab_shard or token_parallel or nvls or graph or lockstep or per_stream or scaled_q" 2>&1 | tail -3
timeout 900 python scripts/sweep_env.py --config llama8b --path fused --reps 4 '' 'LCE_FUSED_GATHER=0'
timeout 900 python scripts/sweep_env.py --config qwen7b --path fused --reps 4 '' 'LCE_FUSED_GATHER=0'
for g in 1 0; do
  for cfg in llama8b llama1b_1m; do
    LCE_FUSED_GATHER=$g timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-split 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('gather=$g $cfg', round(d['value']), round(d['ms_per_step'],2), d['peak_hbm_bytes'])"
  done
done
