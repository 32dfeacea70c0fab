#!/bin/bash
# Launch lists only: tools/gpu_launches.sh TAG "cfgs"   (NCU_CACHE=none for warm-cache, in-situ-like times)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=$1; export TRACE_REPS=1
for c in $2; do
timeout 300 python tools/trace_run.py $c > gpurun_out/trace_${TAG}_c$c.json 2> gpurun_out/trace_${TAG}_c$c.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control ${NCU_CACHE:-all} --csv --log-file gpurun_out/launches_${TAG}_c$c.csv \
    python tools/trace_run.py $c > /dev/null 2>&1; echo "launches c$c rc=$?"
python tools/launch_summary.py gpurun_out/launches_${TAG}_c$c.csv > gpurun_out/launches_${TAG}_c${c}_summary.txt 2>&1
done
