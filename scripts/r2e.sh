python paper_2605_21442_b200/build.py >/dev/null
LCE_DEBUG=1 timeout 600 python -m pytest tests -m gpu -x -q -rs -k "nvls or single_rank or token_parallel or shard or autograd or bf16 or binding" 2>&1 | tail -15
