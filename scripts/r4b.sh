# packed Qwen fused: chunk budget (N_v = 7,177 valid rows: 2 GiB -> 5,632-row chunks, two launches
# per GEMM class and an fp32 dW reduce-add pass; >= 2.49 GB -> one 8,192-row chunk holds every valid row)
python paper_2605_21442_b200/build.py >/dev/null
for rep in 1 2 3; do
  for b in 0 2684354560 4294967296; do
    echo "== qwen7b fused budget $b rep $rep"
    timeout 600 python bench.py --config qwen7b --path fused --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-split --chunk-budget $b 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']), round(d['ms_per_step_median'],3), round(d['peak_hbm_bytes']/1e9,2), d['clocks']['sm_mhz'])"
  done
done
for rep in 1 2; do
  for b in 0 4294967296; do
    echo "== llama70b fused budget $b rep $rep"
    timeout 900 python bench.py --config llama70b --path fused --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-split --chunk-budget $b 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']), round(d['ms_per_step_median'],3), round(d['peak_hbm_bytes']/1e9,2), d['clocks']['sm_mhz'])"
  done
done
