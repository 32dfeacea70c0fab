#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for c in 4 5; do
CMD="python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-brute"
$CMD > gpurun_out/plain_t$c.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:assign_tiles -s 4 -c 1 -o gpurun_out/prof_tiles_c$c $CMD > gpurun_out/ncu_full_t$c.log 2>&1
done
