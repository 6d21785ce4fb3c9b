#!/bin/bash
timeout 1500 python -m pytest tests/test_parity.py -q -m gpu 2>&1 | tail -4
bash scripts/ab_bench.sh ab/liblce_5d0a030.so "llama1b llama8b"
