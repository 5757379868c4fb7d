#!/bin/bash
# Round-2 re-entry session: GPU tests, both bench arms, phase profile, compute-sanitizer.
set -u
O=gpurun_out; mkdir -p $O/sanitizer
timeout 1800 python -m pytest tests -m gpu -q -x > $O/gputest.txt 2>&1; echo "pytest rc=$?" | tee -a $O/gputest.txt
tail -3 $O/gputest.txt
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; cat $O/bench.json
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"; cat $O/bench_ref.json
for c in "512" "64 14336 4096" "64 1024 4096" "64 4096 14336"; do
  echo "== prof $c"; SCB_LIB=scripts/prof_lib.so timeout 300 python scripts/prof_lib.py $c 2>&1 | tail -40
done > $O/prof.txt 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_case.py > $O/sanitizer/$tool.log 2>&1
  echo "$tool rc=$?" | tee -a $O/sanitizer/$tool.log
done
