# binding: per-stream default workspaces (+ autograd / status tests that use them)
python paper_2605_21442_b200/build.py >/dev/null
timeout 900 python -m pytest tests -m gpu -x -q -k "per_stream or autograd or status or bad_label or fused_without_grad or upstream or lockstep" 2>&1 | tail -3
