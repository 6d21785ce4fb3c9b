# round-2 (session 3, final library) ncu evidence (run under gpurun):  bash scripts/prof_r2b.sh
#   launch lists (gpu__time_duration, serialised) of the 8B fused and split steps (2 steps each),
#   --set full of every kernel class of one fused 8B row chunk and of the split path's GEMMs
mkdir -p gpurun_out
python paper_2605_21442_b200/build.py > /dev/null
S="python scripts/one_step.py --config llama8b --steps 2"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/round2c_fused_launches.csv $S --path fused > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/round2c_split_launches.csv $S --path split > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"gemm_|combine_rows|scaled_prep|target_dot|reduce_dh" -c 9 \
    -o gpurun_out/round2c_fused python scripts/one_step.py --config llama8b --path fused > gpurun_out/round2c_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"gemm_" -c 4 \
    -o gpurun_out/round2c_split python scripts/one_step.py --config llama8b --path split >> gpurun_out/round2c_ncu.log 2>&1
tail -n 3 gpurun_out/round2c_ncu.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/round2c_qwen_fused_launches.csv python scripts/one_step.py --config qwen7b --steps 2 --path fused > /dev/null 2>&1
