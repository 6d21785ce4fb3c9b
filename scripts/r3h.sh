# DRAM traffic of the wide dW / dH GEMMs under the K-lockstep drift bound (ncu, one launch each)
python paper_2605_21442_b200/build.py >/dev/null
for cfg in "LCE_LOCK=0" "LCE_LOCK=1 LCE_LOCK_D=64" "LCE_LOCK=1 LCE_LOCK_D=16" "LCE_LOCK=1 LCE_LOCK_D=4"; do
  echo "=== $cfg"
  env $cfg timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct --clock-control none --nvtx --nvtx-include "measure/" --csv \
    python scripts/gemm_power.py --shapes dw,dh --arms wide --seconds 0 --once 2>/dev/null | grep -E '"(dram|gpu__|sm__|lts)' | awk -F'","' '{print $5, $(NF-2), $NF}'
done
