# compute-sanitizer on the final library (K-lockstep in the wide kernels)
python paper_2605_21442_b200/build.py >/dev/null
for tool in memcheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize.py > gpurun_out/round2b_sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/round2b_sanitize_$tool.log
  tail -3 gpurun_out/round2b_sanitize_$tool.log
done
timeout 1500 compute-sanitizer --tool racecheck --print-limit 0 python scripts/sanitize.py 2>&1 | grep -E "Race reported|access at|RACECHECK SUMMARY" | sed -E 's/\+0x[0-9a-f]+//; s/\[[0-9]+ hazards\]//' | sort | uniq -c | sort -rn > gpurun_out/round2b_sanitize_racecheck_summary.log
tail -5 gpurun_out/round2b_sanitize_racecheck_summary.log
