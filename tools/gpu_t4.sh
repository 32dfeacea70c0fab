cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tiles.py -x -q -k "not fullsize" > gpurun_out/t4_pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t4_pytest.txt
bash tools/gpu_ab.sh ${TAG:-br1} "2 1" base v1 v3 v5 v6
