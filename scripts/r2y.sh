LCE_DBG_WAITS=1 LCE_WIDE_2=1 python scripts/one_step.py --config llama8b --path fused --steps 2 2>&1 | grep "lce wide" | head -12
echo "--- fwd wide, pass-2 skipped"
LCE_DBG_WAITS=1 LCE_WIDE_2=1 LCE_DBG_FWD=2 python scripts/one_step.py --config llama8b --path fused --steps 2 2>&1 | grep "lce wide" | head -12
