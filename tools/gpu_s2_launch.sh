#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-x}; C=${2:-5}
python tools/trace_run.py $C > gpurun_out/plain_${TAG}_c$C.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c ${3:-200} --csv --log-file gpurun_out/launches_${TAG}_c$C.csv python tools/trace_run.py $C > /dev/null 2>&1
echo done
