# K-lockstep words via shared-memory atomics: racecheck + timing recheck
python paper_2605_21442_b200/build.py >/dev/null
timeout 900 python -m pytest tests -m gpu -x -q -k "lockstep or wide_schedules or fused_deterministic or debug_gemm" 2>&1 | tail -2
timeout 1500 compute-sanitizer --tool racecheck --print-limit 0 python scripts/sanitize.py 2>&1 | grep -E "Race reported|access at|RACECHECK SUMMARY" | sed -E 's/\+0x[0-9a-f]+//; s/\[[0-9]+ hazards\]//' | sort | uniq -c | sort -rn > gpurun_out/round2b_sanitize_racecheck_summary.log
head -8 gpurun_out/round2b_sanitize_racecheck_summary.log
timeout 900 python scripts/sweep_env.py --config llama8b --path fused --reps 4 '' 'LCE_LOCK=0'
timeout 900 python scripts/sweep_env.py --config llama70b --path fused --reps 2 --steps 3 '' 'LCE_LOCK=0'
