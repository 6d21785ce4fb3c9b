# multi-GPU entry points on a one-GPU box: --gpus 2 must fail loudly; --sweep reports P=1 and skips the rest
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 300 python bench.py --gpus 2 --steps 2 --warmup 3; echo "rc=$?"
timeout 1200 python bench.py --sweep llama8b --steps 3 --warmup 3 2>/dev/null | tail -3; echo "rc=$?"
