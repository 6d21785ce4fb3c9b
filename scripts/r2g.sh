# DRAM traffic of the fused 8B dW / dH / forward GEMMs under L2-hint and raster variants (ncu, cold cache)
python paper_2605_21442_b200/build.py >/dev/null
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
for cfg in "" "LCE_HINT_B_6=2 LCE_HINT_A_6=1" "LCE_HINT_S_6=1" "LCE_HINT_B_6=2 LCE_HINT_A_6=1 LCE_HINT_S_6=1" "LCE_GROUP_M_6=4" "LCE_HINT_B_5=2 LCE_HINT_A_5=1" "LCE_HINT_A_2=2 LCE_HINT_B_2=1"; do
  echo "=== [$cfg]"
  env $cfg timeout 900 ncu --metrics $M --clock-control none -k regex:gemm_ -c 6 --csv python scripts/one_step.py --config llama8b --path fused 2>/dev/null | python scripts/ncu_csv.py

done
timeout 600 python scripts/sweep_env.py --config llama8b --path fused --reps 3 '' 'LCE_DBG_EPI=3' 'LCE_DBG_EPI=4' 'LCE_DBG_EPI=1'
timeout 1500 compute-sanitizer --tool initcheck --print-limit 0 python scripts/sanitize.py 2>&1 | grep -E "^=========\s+at |ERROR SUMMARY|Uninitialized" | sed 's/+0x[0-9a-f]*//' | sort | uniq -c | sort -rn > gpurun_out/initcheck_summary.log
