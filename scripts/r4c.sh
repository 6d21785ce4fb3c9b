# two-chunk default fused budget: fused / full-size parity, default-plan Qwen + 8B bench lines
python paper_2605_21442_b200/build.py >/dev/null
timeout 1500 python -m pytest tests -m gpu -x -q -k "fused or full_size or chunk_budget or random_shapes or kd" 2>&1 | tail -2
for cfg in qwen7b llama8b llama1b; do
  echo "== $cfg fused default"
  timeout 600 python bench.py --config $cfg --path fused --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-split 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']), round(d['ms_per_step_median'],3), round(d['peak_hbm_bytes']/1e9,2), d['clocks']['sm_mhz'], d['roofline']['kernel'], round(d['roofline']['frac'],3))"
done
