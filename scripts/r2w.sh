python paper_2605_21442_b200/build.py >/dev/null
LCE_FWD_ONEPASS=1 LCE_WIDE_2=1 timeout 900 python -m pytest tests -m gpu -x -q -k "fused and not kd and not autograd and not matches_recompute" 2>&1 | tail -2
LCE_FWD_ONEPASS=1 timeout 900 python -m pytest tests -m gpu -x -q -k "fused_tiny or scaled_q or many_row" 2>&1 | tail -2
for cfg in llama8b llama1b; do
timeout 900 python scripts/sweep_env.py --config $cfg --path fused --reps 3 '' 'LCE_FWD_ONEPASS=1' 'LCE_FWD_ONEPASS=1 LCE_WIDE_2=1'
done
timeout 1200 python scripts/sweep_env.py --config llama70b --path fused --reps 2 --steps 3 '' 'LCE_FWD_ONEPASS=1 LCE_WIDE_2=1'
