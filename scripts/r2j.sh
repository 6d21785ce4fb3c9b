bash scripts/prof_r2.sh
bash scripts/all_configs.sh 10 > gpurun_out/round2_all_configs.log 2>&1
timeout 900 python bench.py > gpurun_out/round2_bench.json 2> gpurun_out/round2_bench.err
timeout 1500 python scripts/parity_report.py > gpurun_out/round2_parity_margins.md 2> gpurun_out/parity.err
