# One bench line per BASELINE config and path (1 GPU): the table in BASELINE.md section 5.
#   bash scripts/all_configs.sh [steps]   (+ the fused chunk-budget sweep at 1B / 8B)
STEPS=${1:-10}
summ() {
python -c "
import json, sys
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
r = d['roofline'] or {}
sus, burst = 1368.0, 1629.9
try:
    m = json.load(open('MEASURED_PEAKS.json')); sus, burst = m['bf16_tflops_sustained'], m['bf16_tflops']
except Exception:
    pass
print(json.dumps({'config': d['config']['workload'], 'path': d['path'], 'budget': '$1', 'tok_s': round(d['value']),
  'ms': round(d['ms_per_step'], 2), 'ms_median': round(d['ms_per_step_median'], 2),
  'tensor_frac_sustained': round(d['tensor_frac'], 3), 'tensor_frac_burst': round(d['tensor_frac'] * sus / burst, 3),
  'dom': r.get('kernel'), 'dom_frac': round(r.get('frac', 0), 3), 'dom_util_at_clock': round(r.get('util_at_clock') or 0, 3),
  'peak_hbm_gb': round(d['peak_hbm_bytes'] / 1e9, 2), 'naive_logits_fp32_gb': round(d['naive_logits_bytes_fp32'] / 1e9, 2),
  'sm_mhz': (d['clocks'] or {}).get('sm_mhz'), 'reasons': (d['clocks'] or {}).get('reasons')}))"
}
for cfg in llama1b llama8b qwen7b llama70b llama1b_1m; do
  for path in fused split; do
    echo "== $cfg $path"
    timeout 900 python bench.py --config $cfg --path $path --steps $STEPS --warmup 3 --no-cpu-baseline --no-e2e --no-split 2>/dev/null | summ default
  done
done
for cfg in llama1b llama8b; do
  for b in 536870912 1073741824; do
    echo "== $cfg fused budget $b"
    timeout 600 python bench.py --config $cfg --path fused --steps $STEPS --warmup 3 --no-cpu-baseline --no-e2e --no-split --chunk-budget $b 2>/dev/null | summ $b
  done
done
