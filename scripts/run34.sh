#!/bin/bash
# G TMA store (split path) + AdamW epilogue load hoisting: parity + A/B timing
set -x
timeout 900 python -m pytest tests/test_parity.py -q -m gpu -x 2>&1 | tail -3
timeout 600 python scripts/bench_adamw.py --steps 10 2>&1 | tail -1
for cfg in llama1b llama8b; do
  for z in tma direct; do
    LCE_ZSTORE=$z timeout 300 python bench.py --config $cfg --path split --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', '$z', d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
  done
done
