# K-lockstep drift bound with the 2 us poll (wide D / pair D)
python paper_2605_21442_b200/build.py >/dev/null
timeout 1200 python scripts/sweep_env.py --config llama8b --path fused --reps 4 '' 'LCE_LOCK_D_5=8 LCE_LOCK_D_6=8' 'LCE_LOCK_D_5=32 LCE_LOCK_D_6=32' 'LCE_LOCK_D_2=16' 'LCE_LOCK_D_2=64' 'LCE_LOCK=0'
timeout 1200 python scripts/sweep_env.py --config llama70b --path fused --reps 2 --steps 3 '' 'LCE_LOCK_D_5=8 LCE_LOCK_D_6=8' 'LCE_LOCK_D_2=16' 'LCE_LOCK=0'
