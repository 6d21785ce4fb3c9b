# ncu evidence for one round (run under gpurun):  bash scripts/prof_round.sh <tag>
#   launch lists (gpu__time_duration, serialised) of the 8B fused and split steps,
#   and --set full of every kernel class of one fused 8B row chunk
TAG=${1:-round}
mkdir -p gpurun_out
B="python bench.py --config llama8b --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_fused_launches.csv $B --path fused > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_split_launches.csv $B --path split > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"gemm_|combine_rows|scaled_prep|target_dot|fixup_q|reduce_dh" -c 9 \
    -o gpurun_out/${TAG}_fused python bench.py --config llama8b --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu.log 2>&1
tail -n 2 gpurun_out/${TAG}_ncu.log
