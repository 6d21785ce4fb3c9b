# raster-group sweep: per-kernel ms for several LCE_GROUP_M values (fused and split paths)
for g in 4 8 16 32 64; do
  echo "== fused group $g"; LCE_GROUP_M=$g python bench.py --steps 6 --warmup 2 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
done
for g in 4 8 16 32 64; do
  echo "== split group $g"; LCE_GROUP_M=$g python bench.py --steps 6 --warmup 2 --path split --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
done
