#!/bin/bash
# Launch lists with warm caches (ncu --cache-control none): tools/gpu_launches_warm.sh TAG "cfgs"
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
export TRACE_REPS=1
for c in $2; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/lw_$1_c$c.csv \
    python tools/trace_run.py $c > /dev/null 2>&1; echo "launches c$c rc=$?"
python tools/launch_summary.py gpurun_out/lw_$1_c$c.csv > gpurun_out/lw_$1_c${c}_summary.txt 2>&1
cat gpurun_out/lw_$1_c${c}_summary.txt
done
