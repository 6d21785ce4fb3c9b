# final library: full GPU suite, default bench line, packed-Qwen dW tile-shape A/B at the one-chunk plan
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/round2c_bench_final.json 2> gpurun_out/r4i_bench.err; tail -c 300 gpurun_out/r4i_bench.err
timeout 900 python scripts/sweep_env.py --config qwen7b --path fused --reps 3 '' 'LCE_WIDE_6=0'
