# round1_e: bf16 q chunk + in-place G (fused), TMA G store (split): launch lists, full captures, margins, cuBLAS reference
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r5_fused.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r5_split.csv python bench.py --path split --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"gemm_pair_kernel|fixup_q|combine_rows|reduce_dh" -c 5 -o gpurun_out/prof_r5_fused python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"gemm_pair_kernel" -c 4 -o gpurun_out/prof_r5_split python bench.py --path split --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"gemm_pair_kernel|fixup_q" -c 4 -o gpurun_out/prof_r5_fused1b python bench.py --config llama1b --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 python scripts/parity_report.py > gpurun_out/parity_r5.md 2> gpurun_out/parity_r5.err
timeout 300 python scripts/gemm_vs_cublas.py > gpurun_out/cublas_r5.json 2>&1
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r5.log 2>&1
tail -1 gpurun_out/bench_r5.log | cut -c1-400
