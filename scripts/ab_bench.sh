#!/bin/bash
# A/B: current in-tree liblce.so vs an older build (LCE_LIB_PATH), alternating, same box.
#   bash scripts/ab_bench.sh ab/liblce_<rev>.so "llama1b llama8b" [extra bench args]
OLD=$1; CFGS=$2; shift 2
for rep in 1 2; do
  for cfg in $CFGS; do
    for lib in new old; do
      if [ $lib = old ]; then export LCE_LIB_PATH=$OLD; else unset LCE_LIB_PATH; fi
      timeout 400 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>/dev/null | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$rep $cfg $lib', round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['roofline']['kernel'], d['clocks']['sm_mhz'], d.get('peak_hbm_bytes'))"
    done
  done
done
unset LCE_LIB_PATH
