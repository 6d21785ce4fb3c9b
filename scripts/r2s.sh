for rep in 1 2; do
for P in 4 8; do
  python scripts/bench_shard.py --config llama8b --world $P --rank 0 --steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('P',$P,'no-reserve', d['ms_per_step'], d['bwd_dw'])"
  LCE_VP_RESERVE_TEST=1 python scripts/bench_shard.py --config llama8b --world $P --rank 0 --steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('P',$P,'reserve16 ', d['ms_per_step'], d['bwd_dw'])"
  LCE_VP_RESERVE_TEST=1 LCE_VP_RESERVE_SMS=8 python scripts/bench_shard.py --config llama8b --world $P --rank 0 --steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('P',$P,'reserve8  ', d['ms_per_step'], d['bwd_dw'])"
done
done
