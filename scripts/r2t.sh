python paper_2605_21442_b200/build.py >/dev/null
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
for cfg in "" "LCE_HINT_B_6=2" "LCE_HINT_A_6=2" "LCE_HINT_A_6=2 LCE_HINT_S_6=1" "LCE_HINT_A_5=2" "LCE_HINT_B_5=2"; do
  echo "=== [$cfg]"
  env $cfg timeout 900 ncu --metrics $M --clock-control none -k regex:"gemm_wide" -c 2 --csv python scripts/one_step.py --config llama8b --path fused 2>/dev/null | python scripts/ncu_csv.py
done
timeout 600 python scripts/sweep_env.py --config llama8b --path fused --reps 3 '' 'LCE_HINT_A_6=2' 'LCE_HINT_B_6=2'
