#!/bin/bash
set -u
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/gputest_fast.txt 2>&1; echo "pytest rc=$?"; tail -8 $O/gputest_fast.txt
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; cat $O/bench.json
timeout 1500 python scripts/bench_configs.py > $O/configs.jsonl 2> $O/configs.err; echo "configs rc=$?"; cut -c1-330 $O/configs.jsonl
