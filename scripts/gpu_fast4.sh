#!/bin/bash
set -u
O=gpurun_out; mkdir -p $O
echo "== f64 4096^2 variants"
AB_OPTS="variant=0;variant=16040101" AB_W=128 AB_DTYPE=f64 AB_ROUNDS=2 timeout 300 python scripts/ab_env.py 2>&1 | tail -2
echo "== f64 gate variants"
AB_OPTS="variant=0;variant=16040101" AB_W=32 AB_DTYPE=f64 AB_SHAPE=14336,4096 AB_ROUNDS=2 timeout 300 python scripts/ab_env.py 2>&1 | tail -2
echo "== f32 defaults"
AB_OPTS="variant=0;variant=8040101" AB_W=512 AB_ROUNDS=2 timeout 300 python scripts/ab_env.py 2>&1 | tail -2
AB_OPTS="variant=0;variant=8040101" AB_W=64 AB_SHAPE=14336,4096 AB_ROUNDS=2 timeout 300 python scripts/ab_env.py 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q -x > $O/gputest_fast.txt 2>&1; echo "pytest rc=$?"; tail -8 $O/gputest_fast.txt
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; cat $O/bench.json
