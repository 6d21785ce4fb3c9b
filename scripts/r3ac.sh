# AdamW-in-backward with a coalesced (column-per-lane) state update epilogue: parity + timing
python paper_2605_21442_b200/build.py >/dev/null
timeout 900 python -m pytest tests -m gpu -x -q -k "adamw" 2>&1 | tail -2
for rep in 1 2; do timeout 900 python scripts/bench_adamw.py --config llama8b --steps 10 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:(v['ms_per_step'], v['peak_hbm_gb'], v['kernels_ms']['bwd_dw']) for k,v in d.items()})"; done
