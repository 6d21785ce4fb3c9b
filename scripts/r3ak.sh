# monitor: short naps (prompt exit) + no lockstep in empty launches; forced-lock fallback test, timing recheck
python paper_2605_21442_b200/build.py >/dev/null
LCE_LOCK=1 LCE_LOCK_D=1 timeout 600 python -m pytest tests -m gpu -x -q -k "fallback_rows or lockstep or wide_schedules" 2>&1 | tail -2
timeout 900 python scripts/sweep_env.py --config llama8b --path fused --reps 4 '' 'LCE_LOCK=0'
