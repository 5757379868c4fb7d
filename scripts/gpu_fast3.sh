#!/bin/bash
set -u
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fast_delta or delta" 2>&1 | tail -5
echo "== gate variants"
AB_OPTS="variant=0;variant=16020101;variant=16020201;variant=0|two_phase=1;variant=16020101|two_phase=1" AB_W=64 AB_SHAPE=14336,4096 AB_ROUNDS=2 timeout 300 python scripts/ab_env.py 2>&1 | tail -5
echo "== 4096^2 variants"
AB_OPTS="variant=0;variant=16020101;variant=16020101|two_phase=0;variant=0|two_phase=0" AB_W=512 AB_ROUNDS=2 timeout 300 python scripts/ab_env.py 2>&1 | tail -4
echo "== embed variants"
AB_OPTS="variant=0;variant=16020101;variant=0|two_phase=1" AB_W=64 AB_SHAPE=32000,4096 AB_ROUNDS=2 timeout 300 python scripts/ab_env.py 2>&1 | tail -3
echo "== 1024x4096 variants"
AB_OPTS="variant=0;variant=16020101" AB_W=64 AB_SHAPE=1024,4096 AB_ROUNDS=2 timeout 300 python scripts/ab_env.py 2>&1 | tail -2
