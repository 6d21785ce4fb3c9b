# round1_c profile: final kernels, fused (default bench path) -- launch list + full capture of every kernel class of chunk 0
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r3_fused.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"gemm_pair_kernel|fixup_g|combine_rows|reduce_dh" -c 8 -o gpurun_out/prof_r3_fused python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_r3.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r3_split.csv python bench.py --path split --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 python -m pytest tests/test_parity.py -q -m gpu -k "shard_offsets or full_size" 2>&1 | tail -3
