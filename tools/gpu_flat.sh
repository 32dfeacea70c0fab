#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
O=gpurun_out/flat_bench.txt; : > $O
for rep in 1 2; do
for v in base flat512; do
  L=$PWD/build/var/libkm_$v.so; [ $v = base ] && L=$PWD/paper_2412_02244_b200/libkm.so
  for c in 4 3; do
    r=$(KM_LIB_PATH=$L timeout 200 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-brute 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.readline()); print(d["ms_per_step"])')
    echo "$v c$c $r" >> $O
  done
done
done
