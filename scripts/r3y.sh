# dW under the K-lockstep: H' evict_last with an L2 persisting set-aside (ncu DRAM, fused 8B chunk 0), then in-step A/B
python paper_2605_21442_b200/build.py >/dev/null
for cfg in "LCE_HINT_A_6=0" "LCE_HINT_B_6=2 LCE_L2_PERSIST_MB=80" "LCE_HINT_B_6=2 LCE_L2_PERSIST_MB=100" "LCE_HINT_B_6=2 LCE_HINT_B_5=1 LCE_L2_PERSIST_MB=80"; do
  echo "=== $cfg"
  env $cfg LCE_DEBUG=1 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_wide -c 2 \
    python scripts/one_step.py --config llama8b --path fused 2>&1 | grep -E "gemm_wide|dram__bytes|gpu__time|persisting"
done
timeout 900 python scripts/sweep_env.py --config llama8b --path fused --reps 3 '' 'LCE_HINT_B_6=2 LCE_L2_PERSIST_MB=80'
