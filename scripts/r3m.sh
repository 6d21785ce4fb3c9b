# dW L2 hints under the K-lockstep: G (A) evict_first / H' (B) evict_last -> H' resident across waves?
python paper_2605_21442_b200/build.py >/dev/null
for cfg in "LCE_LOCK=1" "LCE_HINT_A_6=1 LCE_HINT_B_6=2" "LCE_HINT_B_6=2" "LCE_HINT_A_6=1 LCE_HINT_B_6=2 LCE_LOCK_D=8"; do
  echo "=== $cfg"
  env $cfg timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:"EpiDW" -c 2 --csv \
    python scripts/one_step.py --config llama8b --path fused 2>/dev/null | grep -E '"(dram|gpu__|sm__)' | awk -F'","' '{print $(NF-2), $NF}'
done
timeout 900 python scripts/sweep_env.py --config llama8b --path fused --reps 4 '' 'LCE_HINT_A_6=1 LCE_HINT_B_6=2' 'LCE_HINT_B_6=2'
timeout 900 python scripts/sweep_env.py --config llama70b --path fused --reps 2 --steps 3 '' 'LCE_HINT_A_6=1 LCE_HINT_B_6=2'
