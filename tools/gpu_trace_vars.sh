#!/bin/bash
# traces of config $2 for the default lib and build/var variants: tools/gpu_trace_vars.sh TAG CFG VAR...
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=$1; C=$2; shift 2
timeout 300 python tools/trace_run.py $C > gpurun_out/trace_${TAG}_c$C.json 2>&1
for v in "$@"; do KM_LIB_PATH=$PWD/build/var/libkm_$v.so timeout 300 python tools/trace_run.py $C > gpurun_out/trace_${TAG}_${v}_c$C.json 2>&1; done
