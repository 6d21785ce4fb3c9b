#!/bin/bash
# fused CE path with bf16 q chunk (G in place): parity + timing + profile
timeout 900 python -m pytest tests/test_parity.py -q -m gpu -x -k "fused or kd or graph or full or random or smoke" 2>&1 | tail -4
for cfg in llama1b llama8b qwen7b llama70b; do
  timeout 400 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', round(d['value']), d['ms_per_step'], d['roofline'], d['clocks']['sm_mhz'], d.get('peak_hbm_bytes'))"
done
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r5_fused.csv python bench.py --config llama8b --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo ncu rc $?
