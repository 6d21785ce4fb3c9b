# NEXT rows on the final library: reduction none, one-rank vocab-parallel plumbing, KD, AdamW-in-backward; per-rank shard timing
python paper_2605_21442_b200/build.py >/dev/null
timeout 900 python scripts/bench_next.py --config llama8b --steps 10
timeout 900 python scripts/bench_adamw.py --config llama8b --steps 10
timeout 900 python scripts/bench_shard.py 2>&1 | tail -8
