cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bounds.py -x -q > gpurun_out/t5_pytest.txt 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/t5_pytest.txt
for m in auto brute; do
  timeout 600 python bench.py --config 2 --steps 10 --no-cpu-baseline --no-brute --mode $m > gpurun_out/b5_$m.json 2> gpurun_out/b5_$m.err
  python -c "
import json;d=json.load(open('gpurun_out/b5_$m.json'))
print('$m', 'step %.3f'%d['ms_per_step'],'iter %.4f'%d['ms_per_iter'], d['work'] if 'work' in d else '', d.get('roofline',{}).get('assign_ms_per_launch'))" 2>&1 | cut -c1-600
done
