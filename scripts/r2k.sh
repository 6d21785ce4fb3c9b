python paper_2605_21442_b200/build.py >/dev/null
timeout 600 python scripts/sweep_env.py --config llama1b --path fused --reps 3 '' 'LCE_DBG_FWD=1' 'LCE_DBG_FWD=2'
timeout 600 python scripts/sweep_env.py --config llama8b --path fused --reps 3 '' 'LCE_DBG_FWD=1' 'LCE_DBG_FWD=2'
