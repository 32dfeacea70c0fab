#!/bin/bash
# Iteration check: GPU suite, bench lines for the given configs, warm launch lists.
#   tools/gpu_iter.sh TAG "bench cfgs" "launch cfgs" [pytest args]
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/$1; mkdir -p $O
if [ -n "$4" ]; then timeout 1500 python -m pytest tests -m gpu -x -q $4 > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.txt; fi
for c in $2; do
  timeout 600 python bench.py --config $c --steps 10 > $O/bench_config$c.json 2> $O/bench_config$c.err; echo "bench c$c rc=$?"
  python -c "import json;d=json.load(open('$O/bench_config$c.json'));print('c$c', 'ms/iter', round(d['ms_per_iter'],5), 'frac', round(d['roofline']['frac'],3), 'e2e ms/step', round(d['e2e']['ms_per_step'],3))"
done
export TRACE_REPS=1
for c in $3; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file $O/lw_c$c.csv \
    python tools/trace_run.py $c > /dev/null 2>&1; echo "launches c$c rc=$?"
  python tools/launch_summary.py $O/lw_c$c.csv > $O/lw_c${c}_summary.txt 2>&1; cat $O/lw_c${c}_summary.txt
done
