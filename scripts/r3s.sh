# why the K-lockstep slows pair-tile GEMMs: gate vs monitor cost (isolated forward / dW shapes)
python paper_2605_21442_b200/build.py >/dev/null
for cfg in "LCE_LOCK=0" "LCE_LOCK=1 LCE_LOCK_D=16" "LCE_LOCK=1 LCE_LOCK_D=128" "LCE_LOCK=1 LCE_LOCK_D=100000"; do
  echo "=== $cfg"
  env $cfg timeout 300 python scripts/gemm_power.py --shapes fwd,dw --arms pair --seconds 3 | grep -v '^{'
done
timeout 900 python scripts/sweep_env.py --config llama8b --path fused --reps 3 '' 'LCE_LOCK_2=1 LCE_LOCK_D_2=100000' 'LCE_LOCK=0'
