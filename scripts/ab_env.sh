#!/bin/bash
# A/B of an environment knob on the same box, alternating runs:
#   bash scripts/ab_env.sh "LCE_WIDE=1" "llama8b llama1b" [extra bench args]
KNOB=$1; CFGS=$2; shift 2
for rep in 1 2; do
  for cfg in $CFGS; do
    for arm in base knob; do
      if [ $arm = knob ]; then ENVS="$KNOB"; else ENVS=""; fi
      env $ENVS timeout 400 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>/dev/null | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$rep $cfg $arm', round(d['value']), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], ' '.join('%s=%.2f'%(n,v['ms_per_step']) for n,v in k.items() if v['ms_per_step']>0.5))"
    done
  done
done
