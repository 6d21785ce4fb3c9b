# all-config sweep with the K-lockstep (BASELINE.md 5b refresh)
python paper_2605_21442_b200/build.py >/dev/null
bash scripts/all_configs.sh 10 2>&1 | tee gpurun_out/round2b_all_configs.log
