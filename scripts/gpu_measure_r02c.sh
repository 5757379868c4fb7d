#!/bin/bash
# Round-2 final measurements: GPU tests, both bench arms, per-config table, C4 batch (226 x 512), C5, parity shapes
set -u
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/gputest.txt 2>&1; echo "pytest rc=$?"; tail -4 $O/gputest.txt
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; cut -c1-400 $O/bench.json
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"; cut -c1-200 $O/bench_ref.json
timeout 1500 python scripts/bench_configs.py > $O/configs.jsonl 2> $O/configs.err; echo "configs rc=$?"; cut -c1-200 $O/configs.jsonl
timeout 1200 python -m paper_2410_01799_b200.batch --jobs 226 --prefix-cuts 512 --out $O/batch_c4_226x512.json > $O/batch.log 2>&1; echo "batch rc=$?"; tail -3 $O/batch.log | cut -c1-600
timeout 900 python scripts/c5_runs.py > $O/c5_runs.jsonl 2> $O/c5.err; echo "c5 rc=$?"; cut -c1-300 $O/c5_runs.jsonl
timeout 900 python scripts/parity_shapes.py > $O/parity_shapes.txt 2>&1; echo "parity shapes rc=$?"; tail -8 $O/parity_shapes.txt
