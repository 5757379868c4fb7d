#!/bin/bash
# A/B of the barrier-free delta pass (engine option fast_delta) + GPU tests
set -u
O=gpurun_out; mkdir -p $O
AB_OPTS="fast_delta=0;fast_delta=1" AB_W=8 AB_ROUNDS=1 timeout 120 python scripts/ab_env.py 2>&1 | tail -4
echo "w8 rc=$?"
AB_OPTS="fast_delta=0;fast_delta=1" AB_W=64 AB_ROUNDS=2 timeout 180 python scripts/ab_env.py 2>&1 | tail -4
AB_OPTS="fast_delta=0;fast_delta=1" AB_W=512 AB_ROUNDS=3 timeout 300 python scripts/ab_env.py 2>&1 | tail -4
AB_OPTS="fast_delta=0;fast_delta=1" AB_W=256 AB_SHAPE=1024,1024 AB_ROUNDS=3 timeout 300 python scripts/ab_env.py 2>&1 | tail -4
AB_OPTS="fast_delta=0;fast_delta=1" AB_W=64 AB_SHAPE=14336,4096 AB_ROUNDS=2 timeout 300 python scripts/ab_env.py 2>&1 | tail -4
AB_OPTS="fast_delta=0;fast_delta=1" AB_W=64 AB_SHAPE=1024,4096 AB_ROUNDS=2 timeout 300 python scripts/ab_env.py 2>&1 | tail -4
AB_OPTS="fast_delta=0;fast_delta=1" AB_W=64 AB_SHAPE=4096,14336 AB_ROUNDS=2 timeout 300 python scripts/ab_env.py 2>&1 | tail -4
AB_OPTS="fast_delta=0;fast_delta=1" AB_W=128 AB_DTYPE=f64 AB_ROUNDS=2 timeout 300 python scripts/ab_env.py 2>&1 | tail -4
timeout 1500 python -m pytest tests -m gpu -q -x > $O/gputest_fast.txt 2>&1; echo "pytest rc=$?"; tail -15 $O/gputest_fast.txt
