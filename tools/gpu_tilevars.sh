#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for v in A B C D E F; do
  for c in 4 5 3; do
    KM_LIB_PATH=$PWD/build/var/libkm_$v.so timeout 300 python bench.py --config $c --steps 100 --warmup 3 --no-cpu-baseline --no-brute > gpurun_out/tv_${v}_c$c.json 2> gpurun_out/tv_${v}_c$c.err
  done
done
