#!/bin/bash
# tests (default lib), traces for default + variants, section profile (prof lib)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-cmp}; shift
timeout 600 python -m pytest tests/test_gpu_tiles.py tests/test_gpu_dp.py -x -q > gpurun_out/pytest_$TAG.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_$TAG.txt
for c in 4 5 3; do timeout 300 python tools/trace_run.py $c > gpurun_out/trace_${TAG}_c$c.json 2> gpurun_out/trace_${TAG}_c$c.err; done
for v in "$@"; do for c in 4 5 3; do KM_LIB_PATH=$PWD/build/var/libkm_$v.so timeout 300 python tools/trace_run.py $c > gpurun_out/trace_${TAG}_${v}_c$c.json 2> gpurun_out/trace_${TAG}_${v}_c$c.err; done; done
KM_LIB_PATH=$PWD/build/var/libkm_prof.so timeout 300 python tools/prof_tiles.py 4 > gpurun_out/sections_${TAG}_c4.txt 2>&1
echo done
