python paper_2605_21442_b200/build.py >/dev/null
for cfg in llama8b llama70b; do
  steps=10; [ $cfg = llama70b ] && steps=3
  python bench.py --config $cfg --steps $steps --warmup 2 --no-cpu-baseline --no-e2e --no-split | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'config': '$cfg', 'P': 1, 'ms_per_step': d['ms_per_step']}))"
  for P in 2 4 8; do
    LCE_VP_RESERVE_TEST=1 python scripts/bench_shard.py --config $cfg --world $P --rank 0 --steps $steps
  done
done
