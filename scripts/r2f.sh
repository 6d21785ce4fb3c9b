python paper_2605_21442_b200/build.py >/dev/null
for tool in memcheck synccheck racecheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.log
  tail -3 gpurun_out/sanitize_$tool.log
done
