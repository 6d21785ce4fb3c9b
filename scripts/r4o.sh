# full GPU suite after the staging-depth parameterisation; smoke; default bench line
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/round2c_bench_final2.json 2> gpurun_out/r4o_bench.err; tail -c 300 gpurun_out/r4o_bench.err
