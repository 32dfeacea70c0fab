#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
O=gpurun_out/acc4.txt; : > $O
for rep in 1 2; do
for a in "6 1000" "6 10000" "7 1000"; do
  echo "base $a $(timeout 120 python tools/hd_bench.py $a 20 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.readline()); print(d["ms_per_iter"])')" >> $O
  echo "acc4 $a $(KM_LIB_PATH=$PWD/build/var/libkm_acc4.so timeout 120 python tools/hd_bench.py $a 20 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.readline()); print(d["ms_per_iter"])')" >> $O
done
done
KM_LIB_PATH=$PWD/build/var/libkm_acc4.so timeout 400 python -m pytest tests/test_gpu_hd.py -q -m gpu -x > gpurun_out/acc4_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/acc4_pytest.txt
