#!/bin/bash
# A/B of library variants by warm-cache launch lists: tools/gpu_ab_launch.sh TAG "cfgs" KERNEL_REGEX var1 var2 ...
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=$1; CFGS=$2; RX=$3; shift 3
export TRACE_REPS=1
for v in "$@"; do
  for c in $CFGS; do
    case "$v" in base) L="";; *) L=build/var/libkm_$v.so;; esac
    KM_LIB_PATH=$L timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
      --log-file gpurun_out/lw_${TAG}_${v}_c$c.csv python tools/trace_run.py $c > /dev/null 2>&1
    echo "== $v config $c"; python tools/launch_summary.py gpurun_out/lw_${TAG}_${v}_c$c.csv | grep -E "$RX|launches"
  done
done
