#!/bin/bash
# A/B of library variants: tools/gpu_ab.sh TAG "cfgs" var1 var2 ...  (var "base" = the default build)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=$1; CFGS=$2; shift 2
for v in "$@"; do
  for c in $CFGS; do
    EXTRA=""
    case "$v" in st*) EXTRA="--st-shift ${v#st}"; L="";; dbg*) EXTRA="--dbg ${v#dbg}"; L="";; v[0-9]*) EXTRA="--variant ${v#v}"; L="";; base) L="";; *) L=build/var/libkm_$v.so;; esac
    KM_LIB_PATH=$L timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline --no-brute $EXTRA > gpurun_out/ab_${TAG}_${v}_c$c.json 2> gpurun_out/ab_${TAG}_${v}_c$c.err
    python -c "
import sys
import json;d=json.load(open('gpurun_out/ab_${TAG}_${v}_c$c.json'))
print('$v', $c, 'step %.3f'%d['ms_per_step'],'iter %.4f'%d['ms_per_iter'],'K1t %.1f us'%(d['roofline']['assign_ms_per_launch']*1e3),'other/step %.3f'%d['breakdown']['other_ms_per_step'])" >> gpurun_out/ab_${TAG}.txt 2>&1
  done
done
cat gpurun_out/ab_${TAG}.txt
