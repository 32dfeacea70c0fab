cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for v in ${VARS:-1 2 3 4 5 6 7 8}; do for c in 4 2; do
timeout 600 python bench.py --config $c --steps 5 --mode brute --variant $v --no-cpu-baseline --no-brute > gpurun_out/var_$v_$c.json 2>/dev/null
python -c "
import json;d=json.load(open('gpurun_out/var_$v_$c.json'))
r=d['roofline']; print('variant $v config $c', 'K1 %.1f us'%(r['assign_ms_per_launch']*1e3), 'frac %.3f'%r['frac'])"
done; done
