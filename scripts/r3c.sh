# GEMM power/clock: cuBLAS vs our pair / wide mainloops, same shapes and data, back to back
python paper_2605_21442_b200/build.py >/dev/null
timeout 600 python scripts/gemm_power.py --seconds 4
