#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
bash tools/gpu_hd_ncu.sh 6 1000 3
bash tools/gpu_hd_ncu.sh 6 10000 2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hd_gemm -s 2 -c 1 -o gpurun_out/hd_gemm_c6 python tools/hd_bench.py 6 1000 2 > gpurun_out/hd_ncu_full.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hd_certify -s 2 -c 1 -o gpurun_out/hd_certify_c6 python tools/hd_bench.py 6 1000 2 > gpurun_out/hd_ncu_full2.log 2>&1; echo "ncu rc=$?"
