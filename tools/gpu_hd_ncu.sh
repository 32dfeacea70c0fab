#!/bin/bash
# launch list of the high-dimensional path (config $1, k $2, iters $3)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
C=${1:-6}; K=${2:-1000}; I=${3:-3}
timeout 90 python tools/hd_bench.py $C $K $I > gpurun_out/hd_pre_ncu.json 2>&1 || exit 1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/hd_launches_c${C}_k${K}.csv python tools/hd_bench.py $C $K $I > gpurun_out/hd_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/hd_launches_c${C}_k${K}.csv 2>&1 | head -30
