# with the K-lockstep: do wide tiles now pay at shorter K (1B / packed Qwen chunks)?
python paper_2605_21442_b200/build.py >/dev/null
timeout 900 python scripts/sweep_env.py --config llama1b --path fused --reps 4 '' 'LCE_WIDE_6=1' 'LCE_WIDE_5=1' 'LCE_WIDE_5=1 LCE_WIDE_6=1'
timeout 900 python scripts/sweep_env.py --config qwen7b --path fused --reps 4 '' 'LCE_WIDE_6=1' 'LCE_WIDE_5=1 LCE_WIDE_6=1'
timeout 900 python scripts/sweep_env.py --config llama1b --path split --reps 3 '' 'LCE_WIDE_6=1' 'LCE_WIDE_5=1'
