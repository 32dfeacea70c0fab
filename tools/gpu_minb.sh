#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
O=gpurun_out/minb_bench.txt; : > $O
for rep in 1 2; do
for cs in "4 1" "4 2" "3 1" "3 2" "5 1" "5 2" "2 1" "2 2"; do
  set -- $cs
  r=$(KM_K1T_MINB_SEL=$2 timeout 200 python bench.py --config $1 --steps 10 --warmup 3 --no-cpu-baseline --no-brute 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.readline()); print(d["ms_per_step"])')
  echo "c$1 minb$2 $r" >> $O
done
done
