# ncu --set full of the GEMM kernels of one fused 8B row chunk (wide and pair variants)
mkdir -p gpurun_out
B="python bench.py --config llama8b --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
TAG=${1:-wide}
ncu --set full --clock-control none --import-source on -k regex:gemm_ -c 3 -o gpurun_out/prof_$TAG $B > gpurun_out/prof_$TAG.log 2>&1
tail -n 2 gpurun_out/prof_$TAG.log
