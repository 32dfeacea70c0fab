#!/bin/bash
# brute-force path (K1 + privatised update): bench lines for configs 1, 2, 3, 4 in brute mode
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-br}
for c in 1 2 3 4; do
  timeout 600 python bench.py --config $c --steps 10 --mode brute --no-cpu-baseline --no-brute > gpurun_out/brute_${TAG}_c$c.json 2> gpurun_out/brute_${TAG}_c$c.err
  python -c "
import json;d=json.load(open('gpurun_out/brute_${TAG}_c$c.json'))
r=d['roofline']; b=d['breakdown']
print($c, 'step %.3f ms'%d['ms_per_step'],'iter %.4f ms'%d['ms_per_iter'],'K1 %.1f us'%(r['assign_ms_per_launch']*1e3),'frac %.3f'%r['frac'],'fin/iter %.1f us'%(b['finalize_ms_per_iter']*1e3),'other/step %.3f'%b['other_ms_per_step'])" >> gpurun_out/brute_${TAG}.txt 2>&1
done
cat gpurun_out/brute_${TAG}.txt
