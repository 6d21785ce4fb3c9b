# ncu --set full: cuBLAS (fp32 out) vs our wide / pair mainloop on the fused-8B dW / dH shapes, same operands
python paper_2605_21442_b200/build.py >/dev/null
timeout 1200 ncu --set full --clock-control none --nvtx --nvtx-include "measure/" -o gpurun_out/r3e_gemms \
  python scripts/gemm_power.py --shapes dw,dh --arms cublas32,wide,pair --seconds 0 --once > gpurun_out/r3e.txt 2>&1
tail -3 gpurun_out/r3e.txt
timeout 600 python scripts/gemm_power.py --shapes dw,dh --arms cublas32,wide,pair --seconds 3
