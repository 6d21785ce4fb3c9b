python paper_2605_21442_b200/build.py >/dev/null
timeout 600 python scripts/sweep_env.py --config llama8b --path fused --reps 3 '' 'LCE_DW_ACC_PAIR=1'
timeout 900 python scripts/sweep_env.py --config llama70b --path fused --reps 2 --steps 3 '' 'LCE_DW_ACC_PAIR=1'
timeout 600 python scripts/sweep_env.py --config llama1b --path fused --reps 3 '' 'LCE_DW_ACC_PAIR=1'
timeout 1500 compute-sanitizer --tool racecheck --print-limit 0 python scripts/sanitize.py 2>&1 | grep -E "Race reported|access at|RACECHECK SUMMARY" | sed -E 's/\+0x[0-9a-f]+//; s/\[[0-9]+ hazards\]//' | sort | uniq -c | sort -rn > gpurun_out/racecheck_summary.log
