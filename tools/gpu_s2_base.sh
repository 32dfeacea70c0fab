#!/bin/bash
# session-2 baseline: GPU tests, bench at the config's own 20 iterations, launch list
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python bench.py --steps 20 --warmup 3 --no-brute > gpurun_out/bench_c4_20.json 2> gpurun_out/bench_c4_20.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4_20.csv \
  python bench.py --steps 20 --warmup 3 --no-brute --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo done
