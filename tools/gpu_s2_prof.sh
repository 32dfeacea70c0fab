#!/bin/bash
# profile the tile path at config $1 (default 4): plain run, launch list, ncu full of K1t
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
C=${1:-4}
TAG=${2:-v6}
python tools/trace_run.py $C > gpurun_out/plain_$TAG.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_${TAG}_c$C.csv python tools/trace_run.py $C > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:assign_tiles -s 30 -c 1 -o gpurun_out/prof_${TAG}_c$C python tools/trace_run.py $C > gpurun_out/ncu_full_$TAG.log 2>&1
echo done
