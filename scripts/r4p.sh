# phased wide dW schedule (slot-granular ring), A/B only: parity on the debug build first (a lost arrive traps
# instead of hanging), then full-size dW rows and timing on the release build
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
export LCE_WIDE_PHASED=16
LCE_LIB_PATH=$PWD/paper_2605_21442_b200/liblce_debug.so timeout 900 python -m pytest tests -m gpu -x -q -k "wide and (config_shapes or ragged or many_row or chunk_budget or random_shapes or fused)" 2>&1 | tail -3
rc=${PIPESTATUS[0]}
LCE_LIB_PATH=$PWD/paper_2605_21442_b200/liblce_debug.so LCE_WIDE_PHASED=3 timeout 600 python scripts/one_step.py --config llama8b --path fused --steps 1 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -x -q -k "full_size_dweight_rows_and_every_lse and llama8b" 2>&1 | tail -2
unset LCE_WIDE_PHASED
timeout 1200 python scripts/sweep_env.py --config llama8b --path fused --reps 3 '' 'LCE_WIDE_PHASED=16' 'LCE_WIDE_PHASED=8' 'LCE_WIDE_PHASED=0'
