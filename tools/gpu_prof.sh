#!/bin/bash
# Launch list + one full ncu capture of a kernel on a config run (tools/trace_run.py).
#   tools/gpu_prof.sh TAG CONFIG KERNEL_REGEX [SKIP]
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-p}; CFG=${2:-4}; KRE=${3:-assign_tiles}; SKIP=${4:-5}
export TRACE_REPS=1
timeout 300 python tools/trace_run.py $CFG > gpurun_out/trace_$TAG.json 2> gpurun_out/trace_$TAG.err && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python tools/trace_run.py $CFG > /dev/null 2>&1; echo "launches rc=$?"
python tools/launch_summary.py gpurun_out/launches_$TAG.csv > gpurun_out/launches_${TAG}_summary.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KRE -s $SKIP -c 1 \
    -o gpurun_out/ncu_$TAG python tools/trace_run.py $CFG > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu full rc=$?"
