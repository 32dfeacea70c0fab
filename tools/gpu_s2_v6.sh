#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tiles.py tests/test_gpu_dp.py -x -q > gpurun_out/pytest_v6.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_v6.txt
for c in 4 3 2 5; do timeout 300 python tools/trace_run.py $c > gpurun_out/trace_v6_c$c.json 2> gpurun_out/trace_v6_c$c.err; done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_v6_all.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_v6_all.txt
