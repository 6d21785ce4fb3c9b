# K-lockstep with a 2 us monitor poll: which GEMM classes gain (pair tiles too?)
python paper_2605_21442_b200/build.py >/dev/null
ALL="LCE_LOCK=1 LCE_LOCK_D_2=32 LCE_LOCK_D_4=32 LCE_LOCK_D_5=32 LCE_LOCK_D_6=32"
timeout 900 python scripts/sweep_env.py --config llama1b --path fused --reps 4 'LCE_LOCK=0' '' "$ALL"
timeout 900 python scripts/sweep_env.py --config llama8b --path split --reps 3 'LCE_LOCK=0' '' "$ALL"
timeout 900 python scripts/sweep_env.py --config qwen7b --path fused --reps 4 'LCE_LOCK=0' '' "$ALL"
timeout 900 python scripts/sweep_env.py --config llama70b --path fused --reps 2 --steps 3 'LCE_LOCK=0' '' "$ALL"
timeout 900 python scripts/sweep_env.py --config llama8b --path fused --reps 4 'LCE_LOCK=0' '' "$ALL"
