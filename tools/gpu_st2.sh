#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
O=gpurun_out/st2_bench.txt; : > $O
for rep in 1 2; do
for c in 2 1 5 4 3; do
for s in 3 4; do
  r=$(KM_ST_SHIFT=$s timeout 200 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-brute 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.readline()); print(d["ms_per_step"])')
  echo "c$c s$s $r" >> $O
done
done
done
