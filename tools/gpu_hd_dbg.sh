#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for e in 4 12 0; do
for a in "200 128 3 1" "200 256 3 1" "1000 256 7 1" "5000 256 300 1" "3000 64 40 1 grid"; do
  KM_HD_DBG=$e timeout 60 python tools/hd_one.py $a >> gpurun_out/hd_dbg.log 2>&1; echo "[dbg=$e $a] rc=$?" >> gpurun_out/hd_dbg.log
done; done
grep -v "^Traceback\|^  File\|^    " gpurun_out/hd_dbg.log
timeout 900 python -m pytest tests/test_gpu_hd.py -x -q > gpurun_out/hd_tests.log 2>&1; echo "rc=$?" >> gpurun_out/hd_tests.log
tail -3 gpurun_out/hd_tests.log
for c in "6 1000" "7 1000" "6 100" "6 10000" "7 10000"; do timeout 300 python tools/hd_bench.py $c > gpurun_out/hd_bench_$(echo $c | tr ' ' _).json 2>&1; python3 -c "
import json,sys; d=json.loads(open('gpurun_out/hd_bench_$(echo $c | tr ' ' _).json').read().strip().splitlines()[-1]); print(d['config'], d['k'], round(d['ms_per_iter'],3), round(d['gemm_tflops_equiv'],1), d['stats'])" ; done
