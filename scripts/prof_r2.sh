# r2 profile: fused path (default) + split path, launch lists and one full capture per GEMM class
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity.py -q -m gpu 2>&1 | tail -4
python bench.py --steps 10 --warmup 3 --chunk-budget 8589934592 --no-cpu-baseline --no-e2e 2>&1 | tail -1
python bench.py --steps 10 --warmup 3 --path split --no-cpu-baseline --no-e2e 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2_fused.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_pair_kernel -c 4 -o gpurun_out/prof_r2_fused python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_r2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_pair_kernel -c 4 -o gpurun_out/prof_r2_split python bench.py --steps 1 --warmup 0 --path split --no-cpu-baseline --no-e2e > gpurun_out/ncu_r2s.log 2>&1
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r2.log 2>&1
tail -1 gpurun_out/bench_r2.log
