#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for v in 1 2; do
CMD="python bench.py --steps 3 --warmup 3 --variant $v --no-cpu-baseline"
$CMD > gpurun_out/plain_v$v.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:assign_scan -s 2 -c 1 -o gpurun_out/prof_scan_v$v $CMD > gpurun_out/ncu_full_v$v.log 2>&1
done
