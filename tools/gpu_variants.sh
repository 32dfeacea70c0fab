#!/bin/bash
# bench every brute-force scan variant on config 4 (and config 5 for the best ones)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for v in 1 2 3 4 5 6; do
  timeout 300 python bench.py --steps 60 --warmup 5 --variant $v --no-cpu-baseline > gpurun_out/var_c4_v$v.json 2> gpurun_out/var_c4_v$v.err
done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu3.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu3.txt
