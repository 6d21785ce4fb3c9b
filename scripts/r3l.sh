# forward / G raster group with the K-lockstep library (DRAM re-reads of W)
python paper_2605_21442_b200/build.py >/dev/null
timeout 900 python scripts/sweep_env.py --config llama8b --path fused --reps 4 '' 'LCE_GROUP_M_2=32' 'LCE_GROUP_M_2=8'
timeout 900 python scripts/sweep_env.py --config llama8b --path split --reps 3 '' 'LCE_GROUP_M_2=32 LCE_GROUP_M_4=32' 'LCE_GROUP_M_2=64 LCE_GROUP_M_4=64'
