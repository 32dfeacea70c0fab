#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-cfg}
for c in 2 3 5 1; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_${TAG}_c$c.json 2> gpurun_out/bench_${TAG}_c$c.err; done
