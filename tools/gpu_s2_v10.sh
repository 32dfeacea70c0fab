#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-v10}
timeout 600 python -m pytest tests/test_gpu_tiles.py tests/test_gpu_dp.py -x -q > gpurun_out/pytest_$TAG.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_$TAG.txt
for c in 4 5 3 2; do timeout 300 python tools/trace_run.py $c > gpurun_out/trace_${TAG}_c$c.json 2> gpurun_out/trace_${TAG}_c$c.err; done
python tools/trace_run.py 5 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_${TAG}_c5.csv python tools/trace_run.py 5 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_${TAG}_c4.csv python tools/trace_run.py 4 > /dev/null 2>&1
echo done
