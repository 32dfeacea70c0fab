#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 500 python -m pytest tests/test_gpu_dp.py tests/test_gpu_hd.py tests/test_boundary.py -q -m gpu > gpurun_out/pad_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pad_pytest.txt
