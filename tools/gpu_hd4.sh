#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_gpu_hd.py -x -q > gpurun_out/hd_tests.log 2>&1; echo "rc=$?" >> gpurun_out/hd_tests.log
tail -3 gpurun_out/hd_tests.log
for c in "6 1000" "7 1000" "6 100" "6 10000" "7 10000"; do timeout 90 python tools/hd_bench.py $c > gpurun_out/hd_bench_$(echo $c | tr ' ' _).json 2>&1; python3 -c "
import json,sys; d=json.loads(open('gpurun_out/hd_bench_$(echo $c | tr ' ' _).json').read().strip().splitlines()[-1]); print(d['config'], d['k'], round(d['ms_per_iter'],3), round(d['gemm_tflops_equiv'],1), d['stats'])" ; done
bash tools/gpu_hd_ncu.sh 6 1000 3 | grep -i "gemm\|certify\|fallback"
timeout 300 python bench.py --config 6 --steps 5 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_c6.json 2> gpurun_out/bench_c6.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/bench_c6.json
