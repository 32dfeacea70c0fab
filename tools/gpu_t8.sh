cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "expanded or lockstep" > gpurun_out/t8_pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t8_pytest.txt
VARS="2 9 10" bash tools/gpu_brute_ab.sh
CFG=5 VARS="2 9" bash tools/gpu_brute_ab.sh
