# chunk-sized H_c vs the whole-batch H_c (previous library), same box
python paper_2605_21442_b200/build.py >/dev/null
bash scripts/ab_bench.sh ab/liblce_head.so "qwen7b llama8b llama1b" --no-split
