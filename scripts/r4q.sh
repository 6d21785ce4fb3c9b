# phased wide dW, second version (no local-memory arrays in the MMA issue loop): debug-build parity, then timing
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
LCE_WIDE_PHASED=16 LCE_LIB_PATH=$PWD/paper_2605_21442_b200/liblce_debug.so timeout 900 python -m pytest tests -m gpu -x -q -k "wide and (config_shapes or ragged or many_row or fused)" 2>&1 | tail -2
timeout 1200 python scripts/sweep_env.py --config llama8b --path fused --reps 3 '' 'LCE_WIDE_PHASED=0' 'LCE_WIDE_PHASED=16'
