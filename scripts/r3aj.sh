# robustness: the whole GPU suite with the K-lockstep forced on for every GEMM class at the tightest drift bound
python paper_2605_21442_b200/build.py >/dev/null
LCE_LOCK=1 LCE_LOCK_D=1 timeout 600 python -m pytest tests -m gpu -x -q -k "fallback_rows" 2>&1 | grep -E "assert|Error|passed|failed" | head -8
LCE_LOCK=1 LCE_LOCK_D=1 timeout 2400 python -m pytest tests -m gpu -q --deselect "tests/test_parity.py::test_fused_scaled_q_fallback_rows" 2>&1 | tail -3
