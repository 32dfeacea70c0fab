#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:hd_gemm -s 2 -c 1 -o gpurun_out/hd_gemm_c6_v6 python tools/hd_bench.py 6 1000 2 > gpurun_out/hd_ncu_full.log 2>&1; echo "ncu rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:hd_gemm -s 2 -c 1 -o gpurun_out/hd_gemm_c6k1e4_v6 python tools/hd_bench.py 6 10000 2 > gpurun_out/hd_ncu_full2.log 2>&1; echo "ncu rc=$?"
