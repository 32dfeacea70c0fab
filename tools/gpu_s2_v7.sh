#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-v7}
timeout 600 python -m pytest tests/test_gpu_tiles.py tests/test_gpu_dp.py -x -q > gpurun_out/pytest_$TAG.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_$TAG.txt
for c in 4 3 2 5; do timeout 300 python tools/trace_run.py $c > gpurun_out/trace_${TAG}_c$c.json 2> gpurun_out/trace_${TAG}_c$c.err; done
for c in 4 5; do KM_LIB_PATH=$PWD/build/var/libkm_prof.so timeout 300 python tools/prof_tiles.py $c > gpurun_out/sections_${TAG}_c$c.txt 2>&1; done
python tools/trace_run.py 4 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_${TAG}_c4.csv python tools/trace_run.py 4 > /dev/null 2>&1
echo done
