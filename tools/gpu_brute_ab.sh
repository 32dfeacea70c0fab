cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for v in ${VARS:-2 4 6 8}; do
  timeout 600 python bench.py --config ${CFG:-4} --steps 3 --warmup 3 --no-cpu-baseline --no-brute --mode brute --variant $v > gpurun_out/bab_v$v.json 2> gpurun_out/bab_v$v.err
  python -c "
import json;d=json.load(open('gpurun_out/bab_v$v.json'))
r=d['roofline'];print('v$v', 'iter %.4f'%d['ms_per_iter'], 'K1 %.3f ms'%r['assign_ms_per_launch'], 'frac %.3f'%r['frac'])" 2>&1 | tail -1
done
