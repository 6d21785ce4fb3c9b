# AdamW-in-backward: wide vs pair tiles for the AdamW epilogue (26 B/element state RMW)
python paper_2605_21442_b200/build.py >/dev/null
for rep in 1 2; do
for cfg in "LCE_X=0" "LCE_WIDE_6=0" "LCE_WIDE_6=0 LCE_LOCK_6=0"; do
  echo "== $rep $cfg"; env $cfg timeout 900 python scripts/bench_adamw.py --config llama8b --steps 10 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:(v['ms_per_step'], v['peak_hbm_gb'], v['kernels_ms']['bwd_dw']) for k,v in d.items()})"
done
done
