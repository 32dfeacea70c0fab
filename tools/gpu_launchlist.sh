#!/bin/bash
# the recipe's launch-list pass of the bench command (after it exits 0 without ncu)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-brute > gpurun_out/b_ll.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches_bench_c4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-brute > gpurun_out/ncu_ll.log 2>&1; echo "rc=$?"
python tools/launch_summary.py gpurun_out/launches_bench_c4.csv | tail -25
timeout 300 python bench.py --config 6 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b_ll6.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches_bench_c6.csv python bench.py --config 6 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_ll6.log 2>&1; echo "rc=$?"
python tools/launch_summary.py gpurun_out/launches_bench_c6.csv | tail -15
