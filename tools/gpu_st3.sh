#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
O=gpurun_out/st3_bench.txt; : > $O
for rep in 1 2; do
for cs in "4 2" "4 3" "3 2" "3 3" "5 4" "5 5" "2 4" "2 5"; do
  set -- $cs
  r=$(KM_ST_SHIFT=$2 timeout 200 python bench.py --config $1 --steps 10 --warmup 3 --no-cpu-baseline --no-brute 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.readline()); print(d["ms_per_step"])')
  echo "c$1 s$2 $r" >> $O
done
done
KM_ST_SHIFT=2 timeout 300 python -m pytest tests/test_gpu_tiles.py -q -m gpu -x -k "super_tile or full_config4 or equal_brute" > gpurun_out/st3_pytest2.txt 2>&1; echo "rc=$?" >> gpurun_out/st3_pytest2.txt
