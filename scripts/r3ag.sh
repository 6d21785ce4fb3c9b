# fused path with a chunk-sized H_c (gathered per row chunk): parity, time and peak HBM
python paper_2605_21442_b200/build.py >/dev/null
timeout 2000 python -m pytest tests -m gpu -x -q -k "fused or autograd or vocab_shard or token_parallel or nvls or graph or lockstep or per_stream or scaled_q or full_size" 2>&1 | tail -3
for cfg in llama8b llama1b qwen7b llama1b_1m; do
  timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-split 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', round(d['value']), round(d['ms_per_step'],2), d['peak_hbm_bytes'], d['kernels']['gather'])"
done
