# round-2 re-entry: full GPU suite + smoke + default bench line on HEAD
python paper_2605_21442_b200/build.py >/dev/null
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py 2>gpurun_out/r3a_bench.err | tee gpurun_out/r3a_bench.json
