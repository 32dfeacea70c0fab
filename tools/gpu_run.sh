#!/bin/bash
# One gpurun call: GPU test suite (+ optional slow config-5 test), smoke, default bench line.
#   tools/gpu_run.sh TAG [slow] [broken]
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-run}
timeout 1500 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/pytest_gpu_$TAG.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_$TAG.txt
tail -3 gpurun_out/pytest_gpu_$TAG.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$TAG.txt 2>&1; echo "rc=$?" >> gpurun_out/smoke_$TAG.txt
tail -2 gpurun_out/smoke_$TAG.txt
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
if [ "$2" = "slow" ]; then
  KM_SLOW=1 timeout 1500 python -m pytest tests/test_gpu_fullsize.py -k config5 -x -q > gpurun_out/pytest_slow_$TAG.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_slow_$TAG.txt
  tail -2 gpurun_out/pytest_slow_$TAG.txt
fi
if [ "$3" = "broken" ]; then
  # fault injection: Eq. 8 with the radius instead of the diameter must fail the full-size parity
  KM_LIB_PATH=build/var/libkm_broken.so timeout 900 python -m pytest tests/test_gpu_fullsize.py -k "config4 or equal_brute" -q > gpurun_out/pytest_broken_$TAG.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_broken_$TAG.txt
  tail -4 gpurun_out/pytest_broken_$TAG.txt
fi
