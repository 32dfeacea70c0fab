#!/bin/bash
# ncu --set full of one launch of kernel regex $2 at config $1 (skip $3 launches), tag $4
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python tools/trace_run.py $1 > gpurun_out/plain_ncu.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -o gpurun_out/prof_$4 python tools/trace_run.py $1 > gpurun_out/ncu_$4.log 2>&1
echo done
