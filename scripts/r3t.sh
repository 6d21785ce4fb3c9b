# K-lockstep cost on pair tiles: which part (monitor loop / polling / gate atomics)?
python paper_2605_21442_b200/build.py >/dev/null
for v in base m0 m2 s2k; do
  if [ $v = base ]; then unset LCE_LIB_PATH; else export LCE_LIB_PATH=ab/liblce_$v.so; fi
  for cfg in "LCE_LOCK=0" "LCE_LOCK=1 LCE_LOCK_D=100000"; do
    echo "=== $v $cfg"
    env $cfg timeout 300 python scripts/gemm_power.py --shapes fwd --arms pair --seconds 3 | grep -v '^{'
  done
done
