# Qwen packed (N_v 7,177 of 16,384): default chunking (6912 + 265 valid rows) vs a budget that balances the two chunks
python paper_2605_21442_b200/build.py >/dev/null
for rep in 1 2; do
for b in 0 1167851520 1400000000; do
  timeout 600 python bench.py --config qwen7b --path fused --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-split --chunk-budget $b 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$rep budget $b', round(d['value']), round(d['ms_per_step'],3), d['peak_hbm_bytes'], ' '.join('%s=%.2f/%d'%(n,v['ms_per_step'],v['launches_per_step']) for n,v in k.items() if v['ms_per_step']>0.05))"
done
done
