# drop-in API ([B, S, D] hidden, int64 labels) + autograd tests
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "drop_in or autograd or loss_module" 2>&1 | tail -15
