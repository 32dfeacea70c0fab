cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tiles.py -x -q -k "cand_pass" > gpurun_out/t1_pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t1_pytest.txt
bash tools/gpu_ab.sh ${TAG:-cf3} "4 3" base cf2 dbg6=1
