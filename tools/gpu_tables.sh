#!/bin/bash
# ncu --set full tables of the dominant kernel at the other configs (VERDICT r1 missing #6):
# brute K1 at config 4, K1t at configs 3 and 5, K1b at config 2.   tools/gpu_tables.sh TAG
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
export O=gpurun_out/$1; mkdir -p $O
source tools/ncu_cap.sh
export TRACE_REPS=1
cap k1_brute_c4 4 brute assign_scan 3
cap k1b_c2 2 auto bounds_scan 5
cap k1t_c3 3 auto assign_tiles 5
cap k1t_c5 5 auto assign_tiles 3
for n in k1_brute_c4 k1b_c2 k1t_c3 k1t_c5; do
  zcat $O/ncu_${n}_source.csv.gz > /tmp/src.csv; python tools/ncu_lines.py /tmp/src.csv 30 > $O/ncu_${n}_lines.txt 2>&1
  rm -f $O/ncu_${n}_source.csv.gz $O/ncu_${n}_raw.csv.gz
done
