#!/bin/bash
# ncu --set full of the dominant kernels at config 4: K1t (tile path, an iteration ~10 of the
# 2nd run) and K1 (brute force), for the roofline "traffic" field
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-roof}
python tools/trace_run.py 4 > gpurun_out/plain_roof.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:assign_tiles -s 30 -c 1 -o gpurun_out/prof_${TAG}_k1t python tools/trace_run.py 4 > gpurun_out/ncu_${TAG}_k1t.log 2>&1
python tools/trace_run.py 4 brute > gpurun_out/plain_roof_b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:assign_fast -s 5 -c 1 -o gpurun_out/prof_${TAG}_k1 python tools/trace_run.py 4 brute > gpurun_out/ncu_${TAG}_k1.log 2>&1
echo done
