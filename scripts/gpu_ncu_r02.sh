#!/bin/bash
# Round-2 ncu evidence (one gpurun call; every ncu command is preceded by the same
# command run plainly, exiting 0).  Outputs in gpurun_out/; summarised into
# profiles/r02/ by scripts/ncu_summary.py.
set -u
O=gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/plain_bench.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1
echo "launch list rc=$?"
python scripts/prof_case.py 512 > $O/plain_512.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -o $O/sweep_bench512 \
      python scripts/prof_case.py 512 > $O/ncu_512.log 2>&1
echo "bench kernel full rc=$?"
python scripts/prof_case.py 16 14336 4096 > $O/plain_gate.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -o $O/sweep_gate16 \
      python scripts/prof_case.py 16 14336 4096 > $O/ncu_gate.log 2>&1
echo "gate full rc=$?"
python scripts/prof_case.py 1 c5 > $O/plain_c5.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -o $O/sweep_c5 \
      python scripts/prof_case.py 1 c5 > $O/ncu_c5.log 2>&1
echo "c5 full rc=$?"
ls -la $O
