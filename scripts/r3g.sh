# K-lockstep with a monitor warp: parity, then A/B per class and drift bound
python paper_2605_21442_b200/build.py >/dev/null
timeout 900 python -m pytest tests -m gpu -x -q -k "debug_gemm or fused_many or random_shapes or tiny_config or fused_config_shapes or graph" 2>&1 | tail -2
LCE_LOCK=1 timeout 600 python scripts/gemm_power.py --shapes dw,dh --arms wide,pair --seconds 3 | grep -v '^{'
LCE_LOCK=0 timeout 600 python scripts/gemm_power.py --shapes dw,dh --arms wide,pair --seconds 3 | grep -v '^{'
timeout 900 python scripts/sweep_env.py --config llama8b --path fused --reps 3 '' 'LCE_LOCK=0' 'LCE_LOCK=1' 'LCE_LOCK_D=16' 'LCE_LOCK_D=32' 'LCE_LOCK_D=128'
timeout 900 python scripts/sweep_env.py --config llama8b --path split --reps 3 '' 'LCE_LOCK=0' 'LCE_LOCK=1' 'LCE_LOCK_D=32'
