#!/bin/bash
# Alternating A/B/C... of environment settings on one box:
#   bash scripts/ab_multi.sh "llama8b llama1b" "" "LCE_WIDE=0" "LCE_WIDE_LAG=1" -- [extra bench args]
CFGS=$1; shift
ARMS=()
while [ $# -gt 0 ] && [ "$1" != "--" ]; do ARMS+=("$1"); shift; done
[ "$1" = "--" ] && shift
for rep in 1 2; do
  for cfg in $CFGS; do
    for arm in "${ARMS[@]}"; do
      env $arm timeout 400 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>/dev/null | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$rep $cfg [$arm]', round(d['value']), round(d['ms_per_step'],3), (d.get('clocks') or {}).get('sm_mhz'), ' '.join('%s=%.2f%s'%(n,v['ms_per_step'],('@%d/%.3f'%(v['sm_mhz'],v['util_at_clock'])) if 'util_at_clock' in v else '') for n,v in k.items() if v['ms_per_step']>0.3))"
    done
  done
done
