# final-library evidence: ncu launch lists + --set full (8B both paths, Qwen fused launch list), all-config sweep
python paper_2605_21442_b200/build.py >/dev/null
bash scripts/prof_r2c.sh
bash scripts/all_configs.sh 10 > gpurun_out/round2c_all_configs.log 2>&1
