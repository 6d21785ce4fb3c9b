# KD (NEXT-4) step time / peak HBM vs chunk budget, 8B student + same-shape teacher
python paper_2605_21442_b200/build.py >/dev/null
timeout 900 python scripts/kd_budget.py
