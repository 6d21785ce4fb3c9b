# full GPU suite + smoke + default bench with the K-lockstep on wide tiles
python paper_2605_21442_b200/build.py >/dev/null
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py 2>gpurun_out/r3j_bench.err | tee gpurun_out/r3j_bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['roofline'], d['split']['value'], d['split']['roofline']['frac'])"
