cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for cm in "2 tiles" "2 bounds" "3 bounds" "3 tiles" "4 bounds" "5 bounds"; do
  set -- $cm
  timeout 600 python bench.py --config $1 --steps 5 --warmup 3 --no-cpu-baseline --no-brute --mode $2 > gpurun_out/md_$1_$2.json 2> gpurun_out/md_$1_$2.err
  python -c "
import json;d=json.load(open('gpurun_out/md_$1_$2.json'))
print('c$1 $2', 'iter %.4f ms'%d['ms_per_iter'], 'scanned/iter', d['work']['points_scanned_per_iter'])" 2>&1 | tail -1
done
