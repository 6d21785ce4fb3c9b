python paper_2605_21442_b200/build.py >/dev/null
timeout 900 python -m pytest tests -m gpu -x -q -k "fused or scaled_q or autograd or random_shapes or token_parallel" 2>&1 | tail -3
timeout 600 python scripts/sweep_env.py --config llama1b --path fused --reps 3 '' 'LCE_FWD_ONEPASS=0'
timeout 600 python scripts/sweep_env.py --config llama8b --path fused --reps 3 '' 'LCE_FWD_ONEPASS=0'
timeout 900 python bench.py > gpurun_out/bench_r2d.json 2> gpurun_out/bench_r2d.err; tail -c 3000 gpurun_out/bench_r2d.json
