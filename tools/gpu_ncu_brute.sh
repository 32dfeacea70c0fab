#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=$1; CFG=${2:-4}
export TRACE_REPS=1
timeout 300 python tools/trace_run.py $CFG brute > gpurun_out/trace_$TAG.json 2> gpurun_out/trace_$TAG.err && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:assign_scan -s 3 -c 1 \
    -o gpurun_out/ncu_$TAG python tools/trace_run.py $CFG brute > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu rc=$?"
