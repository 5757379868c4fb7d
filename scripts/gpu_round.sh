#!/bin/bash
# One GPU-box session: parity tests, bench, then (only if the bench exited 0)
# the ncu launch list of the same command and one --set full capture of the
# sweep kernel.  Everything lands in gpurun_out/ (copy summaries to profiles/).
# usage: scripts/gpu_round.sh [tag] [skip-tests]
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
if [ "${2:-}" != "skip-tests" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x > $OUT/gputest_$TAG.txt 2>&1
  echo "pytest rc=$?" >> $OUT/gputest_$TAG.txt
fi
timeout 600 python bench.py --steps 5 --warmup 3 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
rc=$?
echo "bench rc=$rc"
if [ $rc -eq 0 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > $OUT/ncu_launch_$TAG.log 2>&1
  echo "ncu launches rc=$?"
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:sweep_kernel -c 1 \
    -o $OUT/sweep_$TAG python bench.py --steps 1 --warmup 0 --no-cpu-baseline \
    > $OUT/ncu_full_$TAG.log 2>&1
  echo "ncu full rc=$?"
fi
