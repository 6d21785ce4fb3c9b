timeout 900 python scripts/sweep_env.py --config llama8b --path fused --reps 3 '' 'LCE_WIDE_2=1' 'LCE_WIDE_2=1 LCE_DBG_FWD=2' 'LCE_DBG_FWD=2'
