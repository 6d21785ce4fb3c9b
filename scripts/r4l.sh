# parity margins of the final library (two-chunk fused plan) vs the fp64 oracle
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 2400 python scripts/parity_report.py > gpurun_out/round2c_parity_margins.md 2> gpurun_out/r4l.err
tail -3 gpurun_out/r4l.err
