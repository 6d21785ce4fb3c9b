# K-lockstep monitor poll period: 256 ns (base) vs 1 / 2 / 4 us, wide-only default and with the forward locked
python paper_2605_21442_b200/build.py >/dev/null
for rep in 1 2; do
for v in base s1k s2k s4k; do
  if [ $v = base ]; then unset LCE_LIB_PATH; else export LCE_LIB_PATH=ab/liblce_$v.so; fi
  for cfg in "LCE_LOCK=0" "" "LCE_LOCK_2=1 LCE_LOCK_D_2=32"; do
    env $cfg timeout 400 python bench.py --config llama8b --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-split 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$rep $v [$cfg]', round(d['value']), round(d['ms_per_step'],3), ' '.join('%s=%.2f@%d'%(n,v['ms_per_step'],v.get('sm_mhz') or 0) for n,v in k.items() if v['ms_per_step']>1))"
  done
done
done
