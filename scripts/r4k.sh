# fused plan: row buffers bounded by the budget (small V); fused / full-size parity; 8B + Qwen fused bench unchanged
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -k "fused or full_size or chunk_budget or kd" 2>&1 | tail -2
for cfg in llama8b qwen7b; do
  timeout 600 python bench.py --config $cfg --path fused --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-split 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$cfg', round(d['value']), round(d['ms_per_step_median'],3), round(d['peak_hbm_bytes']/1e9,2))"
done
