#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-s}
for c in 4 5; do KM_LIB_PATH=$PWD/build/var/libkm_prof.so timeout 300 python tools/prof_tiles.py $c > gpurun_out/sections_${TAG}_c$c.txt 2>&1; done
