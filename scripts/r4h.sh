# debug build (trapping spin-wait timeouts): the debug-sync GPU test + smoke on the release build
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
ls -la paper_2605_21442_b200/*.so
timeout 1200 python -m pytest tests -m gpu -x -q -k "debug_sync or tiny_config or fused_tiny" 2>&1 | tail -3
