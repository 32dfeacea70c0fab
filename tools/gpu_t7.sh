cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bounds.py tests/test_boundary.py -x -q > gpurun_out/t7_pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t7_pytest.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/t7_smoke.txt 2>&1; echo "smoke rc=$?"
for c in 1 2; do
  timeout 600 python bench.py --config $c --steps 20 --no-cpu-baseline --no-brute > gpurun_out/b7_c$c.json 2> gpurun_out/b7_c$c.err
  python -c "
import json;d=json.load(open('gpurun_out/b7_c$c.json'))
print($c, 'step %.4f'%d['ms_per_step'],'iter %.4f'%d['ms_per_iter'], 'e2e', d['e2e']['ms_per_step'])"
done
