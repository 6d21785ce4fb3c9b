# NVTX ranges: ncu filtered by the lce_forward_backward range and by a step range; smoke; bench (overhead check)
python paper_2605_21442_b200/build.py >/dev/null
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
ncu --nvtx --nvtx-include "lce_forward_backward/" --metrics gpu__time_duration.sum -c 6 python scripts/one_step.py --config llama1b --path fused --steps 1 2>&1 | grep -E "gemm_|kernel|NVTX|==PROF==" | head -20
ncu --nvtx --nvtx-include "lce_forward_backward/S5 dW GEMM/" --metrics gpu__time_duration.sum -c 4 python scripts/one_step.py --config llama1b --path fused --steps 1 2>&1 | grep -E "gemm_|==PROF==" | head -10
timeout 600 python bench.py --no-cpu-baseline --no-split 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']), round(d['ms_per_step_median'],3), d['e2e']['value'], d['clocks'])"
