# ncu --set full of cuBLAS's kernels on the fused 8B chunk shapes (reference for our GEMMs)
mkdir -p gpurun_out
cat > /tmp/cub1.py <<'PY'
import torch
g = torch.Generator(device="cuda").manual_seed(0)
H = torch.randn(8192, 4096, device="cuda", generator=g).bfloat16()
W = (torch.randn(128256, 4096, device="cuda", generator=g) / 64).bfloat16()
G = (torch.randn(8192, 128256, device="cuda", generator=g) * 1e-5).bfloat16()
for _ in range(2):
    torch.matmul(H, W.t()); torch.matmul(G, W); torch.matmul(G.t(), H)
torch.cuda.synchronize()
PY
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cublas_launches.csv python /tmp/cub1.py > /dev/null 2>&1
ncu --set full --clock-control none -k regex:"nvjet|gemm|Kernel|sm100|cutlass" -s 3 -c 3 -o gpurun_out/prof_cublas python /tmp/cub1.py > gpurun_out/prof_cublas.log 2>&1
tail -3 gpurun_out/prof_cublas.log
