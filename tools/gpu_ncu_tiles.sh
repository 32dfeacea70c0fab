#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tiles.py -x -q > gpurun_out/pytest_tiles.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_tiles.txt
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-brute"
$CMD > gpurun_out/plain_t.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_tiles.csv $CMD > gpurun_out/ncu_launches_t.log 2>&1
$CMD > gpurun_out/plain_t2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:assign_tiles -s 4 -c 1 -o gpurun_out/prof_tiles $CMD > gpurun_out/ncu_full_t.log 2>&1
