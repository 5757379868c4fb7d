set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_around_gpu.py -q -x > gpurun_out/around_gpu.txt 2>&1; echo "around rc=$?" >> gpurun_out/around_gpu.txt
timeout 600 python scripts/bench_around.py > gpurun_out/bench_around.jsonl 2> gpurun_out/bench_around.err; echo "bench_around rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:expand_kernel -c 1 -o gpurun_out/expand_r01 python scripts/bench_around.py --only expand --steps 1 --no-cpu > gpurun_out/ncu_expand.log 2>&1; echo "ncu rc=$?"
timeout 900 python -m pytest tests -q -x -m gpu > gpurun_out/gputest_all.txt 2>&1; echo "all rc=$?" >> gpurun_out/gputest_all.txt
