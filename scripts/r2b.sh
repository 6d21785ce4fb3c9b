python paper_2605_21442_b200/build.py >/dev/null
timeout 600 python scripts/sweep_env.py --config llama8b --path fused --reps 3 '' 'LCE_DBG_EPI=1' 'LCE_DBG_EPI=2' 'LCE_WIDE_6=0'
timeout 600 python scripts/sweep_env.py --config llama8b --path split --reps 2 '' 'LCE_DBG_EPI=1' 'LCE_DBG_EPI=2' 'LCE_WIDE_6=0'
