#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
CMD="python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline --no-brute"
$CMD > gpurun_out/plain_t4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:assign_tiles -s 4 -c 1 -o gpurun_out/prof_tiles5_c4 $CMD > gpurun_out/ncu_full_t4.log 2>&1
ncu -i gpurun_out/prof_tiles5_c4.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_tiles5_src.csv 2>&1
