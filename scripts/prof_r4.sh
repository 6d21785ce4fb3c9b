# round1_d: final kernels (TMA Z store): launch lists at 8B (fused, split) and 1B (fused), full capture of the fused 8B chunk
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r4_fused.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r4_split.csv python bench.py --path split --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"gemm_pair_kernel|fixup_g|combine_rows|reduce_dh" -c 6 -o gpurun_out/prof_r4_fused python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"gemm_pair_kernel" -c 4 -o gpurun_out/prof_r4_split python bench.py --path split --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"gemm_pair_kernel" -c 3 -o gpurun_out/prof_r4_fused1b python bench.py --config llama1b --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r4.log 2>&1
tail -1 gpurun_out/bench_r4.log | cut -c1-300
