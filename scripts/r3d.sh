# mbarrier wait variants (suspend-time hints / sleep backoff): GEMM clock at equal power, then the 8B step
python paper_2605_21442_b200/build.py >/dev/null
for rep in 1 2; do
for v in base v1 v2 v3; do
  if [ $v = base ]; then unset LCE_LIB_PATH; else export LCE_LIB_PATH=ab/liblce_$v.so; fi
  echo "== $rep $v"
  timeout 300 python scripts/gemm_power.py --shapes dh,dw --arms pair,wide --seconds 3 2>&1 | grep -v '^{'
done
done
unset LCE_LIB_PATH
for rep in 1 2; do
for v in base v1 v2 v3; do
  if [ $v = base ]; then unset LCE_LIB_PATH; else export LCE_LIB_PATH=ab/liblce_$v.so; fi
  timeout 400 python bench.py --config llama8b --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$rep $v', round(d['value']), round(d['ms_per_step'],3), (d.get('clocks') or {}).get('sm_mhz'), ' '.join('%s=%.2f%s'%(n,v['ms_per_step'],('@%d/%.3f'%(v['sm_mhz'],v['util_at_clock'])) if 'util_at_clock' in v else '') for n,v in k.items() if v['ms_per_step']>0.3))"
done
done
