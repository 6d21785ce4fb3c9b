# One bench line per BASELINE config and path (1 GPU): the table in BASELINE.md section 5.
for cfg in llama1b llama8b qwen7b llama70b llama1b_1m; do
  for path in fused split; do
    echo "== $cfg $path"
    timeout 600 python bench.py --config $cfg --path $path --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json, sys
d = json.loads(sys.stdin.read())
r = d['roofline'] or {}
print(json.dumps({'config': d['config']['workload'], 'path': d['path'], 'tok_s': round(d['value']), 'ms': round(d['ms_per_step'], 2),
  'tensor_frac': round(d['tensor_frac'], 3), 'dom': r.get('kernel'), 'dom_frac': round(r.get('frac', 0), 3),
  'peak_hbm_gb': round(d['peak_hbm_bytes'] / 1e9, 2), 'naive_logits_fp32_gb': round(d['naive_logits_bytes_fp32'] / 1e9, 2),
  'sm_mhz': (d['clocks'] or {}).get('sm_mhz')}))"
  done
done
