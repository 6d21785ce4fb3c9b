# compute-sanitizer on the final library (round 2 session 3: dH slab TMA stores, two-chunk plan)
python paper_2605_21442_b200/build.py >/dev/null
timeout 900 python -m pytest tests -m gpu -x -q -k "default_plan_chunk_boundary" 2>&1 | tail -2
for tool in memcheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize.py > gpurun_out/round2c_sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/round2c_sanitize_$tool.log
  tail -3 gpurun_out/round2c_sanitize_$tool.log
done
timeout 1500 compute-sanitizer --tool racecheck --print-limit 0 python scripts/sanitize.py 2>&1 | grep -E "Race reported|access at|RACECHECK SUMMARY" | sed -E 's/\+0x[0-9a-f]+//; s/\[[0-9]+ hazards\]//' | sort | uniq -c | sort -rn > gpurun_out/round2c_sanitize_racecheck_summary.log
tail -5 gpurun_out/round2c_sanitize_racecheck_summary.log
