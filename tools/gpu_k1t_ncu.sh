#!/bin/bash
# one ncu --set full capture of K1t (config 4, an iteration in the middle of a run) -> DRAM traffic
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TRACE_REPS=1 timeout 300 python tools/trace_run.py 4 > /dev/null 2>&1 || exit 1
TRACE_REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:assign_tiles_kernel -s 10 -c 1 -o gpurun_out/k1t_c4_final python tools/trace_run.py 4 > /dev/null 2>&1; echo "rc=$?"
