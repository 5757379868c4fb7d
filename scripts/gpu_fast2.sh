#!/bin/bash
# fast_delta A/B on the main shapes, phase profile, then the GPU tests
set -u
O=gpurun_out; mkdir -p $O
AB_OPTS="fast_delta=0;fast_delta=1" AB_W=8 AB_ROUNDS=1 timeout 120 python scripts/ab_env.py 2>&1 | tail -2
AB_OPTS="fast_delta=0;fast_delta=1" AB_W=512 AB_ROUNDS=2 timeout 300 python scripts/ab_env.py 2>&1 | tail -2
AB_OPTS="fast_delta=0;fast_delta=1" AB_W=256 AB_SHAPE=1024,1024 AB_ROUNDS=2 timeout 300 python scripts/ab_env.py 2>&1 | tail -2
AB_OPTS="fast_delta=0;fast_delta=1" AB_W=64 AB_SHAPE=14336,4096 AB_ROUNDS=2 timeout 300 python scripts/ab_env.py 2>&1 | tail -2
AB_OPTS="fast_delta=0;fast_delta=1" AB_W=64 AB_SHAPE=1024,4096 AB_ROUNDS=2 timeout 300 python scripts/ab_env.py 2>&1 | tail -2
AB_OPTS="fast_delta=0;fast_delta=1" AB_W=64 AB_SHAPE=4096,14336 AB_ROUNDS=2 timeout 300 python scripts/ab_env.py 2>&1 | tail -2
AB_OPTS="fast_delta=0;fast_delta=1" AB_W=64 AB_SHAPE=32000,4096 AB_ROUNDS=2 timeout 300 python scripts/ab_env.py 2>&1 | tail -2
AB_OPTS="fast_delta=0;fast_delta=1" AB_W=128 AB_DTYPE=f64 AB_ROUNDS=2 timeout 300 python scripts/ab_env.py 2>&1 | tail -2
for c in "512" "256 1024 1024" "64 14336 4096"; do SCB_LIB=scripts/prof_lib.so timeout 200 python scripts/prof_lib.py $c 2>&1 | grep -E "fast delta|prof matrix|prof3|kernel_ms"; done
if [ "${1:-}" != "notests" ]; then
timeout 1500 python -m pytest tests -m gpu -q -x > $O/gputest_fast.txt 2>&1; echo "pytest rc=$?"; tail -8 $O/gputest_fast.txt
fi
