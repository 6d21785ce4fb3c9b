timeout 1500 python -m pytest tests/test_parity.py -q -m gpu -x 2>&1 | tail -3
bash scripts/ab_bench.sh ab/liblce_6c4fe69.so "llama1b llama8b"
bash scripts/ab_bench.sh ab/liblce_6c4fe69.so "llama8b" --path split
