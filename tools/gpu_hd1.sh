#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_hd.py -x -q > gpurun_out/hd_tests.log 2>&1; echo "rc=$?" >> gpurun_out/hd_tests.log
tail -5 gpurun_out/hd_tests.log
for c in "6 1000" "7 1000" "6 100" "6 10000"; do timeout 300 python tools/hd_bench.py $c > gpurun_out/hd_bench_$(echo $c | tr ' ' _).json 2>&1; tail -c 700 gpurun_out/hd_bench_$(echo $c | tr ' ' _).json; echo; done
