#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
bash tools/gpu_tiles.sh
for c in 4 5 3; do KM_LIB_PATH=$PWD/build/var/libkm_prof.so python tools/prof_tiles.py $c > gpurun_out/prof_sections_c$c.txt 2>&1; done
