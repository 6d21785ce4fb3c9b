python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 2700 python -m pytest tests -m gpu -q -x -rs --durations=10 2>&1 | tail -25
