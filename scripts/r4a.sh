# session 3 re-entry: full GPU suite + smoke + default bench line at HEAD
mkdir -p gpurun_out
python paper_2605_21442_b200/build.py >/dev/null
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/r4a_bench.json 2> gpurun_out/r4a_bench.err; tail -c 400 gpurun_out/r4a_bench.err
