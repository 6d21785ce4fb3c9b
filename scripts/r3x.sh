# final-library check: full GPU suite, smoke, default bench line, then ncu evidence (prof_r2b)
python paper_2605_21442_b200/build.py >/dev/null
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py 2>gpurun_out/r3x_bench.err > gpurun_out/r3x_bench.json; python -c "import json; d=json.load(open('gpurun_out/r3x_bench.json')); print(d['value'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['util_at_clock'], d['split']['value'], d['clocks'])"
bash scripts/prof_r2b.sh
