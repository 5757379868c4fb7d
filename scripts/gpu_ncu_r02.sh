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
# summaries on the box (the reports are ~24 MB each; gpurun brings back <= 64 MiB)
mkdir -p $O/r02
python scripts/ncu_summary.py --rep $O/sweep_bench512.ncu-rep --out $O/r02/sweep_kernel_bench512_full.txt \
  --desc "python scripts/prof_case.py 512 (the bench workload: 4096^2 f32, 512 cuts, seed 1)" --cuts 512 \
  --launches $O/launches_bench.csv --traffic > /dev/null 2>&1; echo "summary bench rc=$?"
python scripts/ncu_summary.py --rep $O/sweep_gate16.ncu-rep --out $O/r02/sweep_kernel_gate16_full.txt \
  --desc "python scripts/prof_case.py 16 14336 4096 (C4 gate shape, HBM-resident, 16 cuts)" --cuts 16 > /dev/null 2>&1
python scripts/ncu_summary.py --rep $O/sweep_c5.ncu-rep --out $O/r02/sweep_kernel_c5_full.txt \
  --desc "python scripts/prof_case.py 1 c5 (C5 65536^2 f32, 1 cut)" --cuts 1 > /dev/null 2>&1
for x in bench512 gate16 c5; do python scripts/ncu_hotlines.py $O/sweep_$x.ncu-rep 40 > $O/r02/hotlines_$x.txt 2>&1; done
cp profiles/latest_kernel_traffic.json $O/r02/ 2>/dev/null  # written just above by --traffic
rm -f $O/sweep_gate16.ncu-rep $O/sweep_c5.ncu-rep $O/sweep_bench512.ncu-rep
ls -la $O/r02
