# K-lockstep in the step: drift bound and per-class A/B, more reps
python paper_2605_21442_b200/build.py >/dev/null
timeout 1200 python scripts/sweep_env.py --config llama8b --path fused --reps 5 'LCE_LOCK=0' 'LCE_LOCK_D=16' 'LCE_LOCK_D=8' 'LCE_LOCK_D=16 LCE_LOCK_2=1'
timeout 900 python scripts/sweep_env.py --config llama8b --path split --reps 4 'LCE_LOCK=0' 'LCE_LOCK_D=16' 'LCE_LOCK_D=16 LCE_LOCK_2=1 LCE_LOCK_4=1'
timeout 900 python scripts/sweep_env.py --config llama70b --path fused --reps 2 --steps 4 'LCE_LOCK=0' 'LCE_LOCK_D=16'
timeout 900 python scripts/sweep_env.py --config llama1b --path fused --reps 4 'LCE_LOCK=0' 'LCE_LOCK_D=16'
