# K-lockstep on the pair-tile forward / G GEMMs with a looser drift bound
python paper_2605_21442_b200/build.py >/dev/null
timeout 1200 python scripts/sweep_env.py --config llama8b --path fused --reps 4 '' 'LCE_LOCK_2=1 LCE_LOCK_D_2=32' 'LCE_LOCK_2=1 LCE_LOCK_D_2=64' 'LCE_LOCK_2=1 LCE_LOCK_D_2=128'
timeout 900 python scripts/sweep_env.py --config llama8b --path split --reps 3 '' 'LCE_LOCK_2=1 LCE_LOCK_4=1 LCE_LOCK_D_2=64 LCE_LOCK_D_4=64'
timeout 900 python scripts/sweep_env.py --config llama1b --path fused --reps 4 '' 'LCE_LOCK_2=1 LCE_LOCK_D_2=64' 'LCE_LOCK_6=1 LCE_LOCK_D_6=64' 'LCE_LOCK_5=1 LCE_LOCK_D_5=64'
