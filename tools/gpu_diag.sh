#!/bin/bash
# Diagnostic captures: ncu --set full with source for the candidate pass and K1t at a config.
#   tools/gpu_diag.sh TAG CONFIG
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
export O=gpurun_out/$1; mkdir -p $O
C=${2:-4}
timeout 600 python -m pytest tests -m gpu -x -q tests/test_gpu_tiles.py > $O/pytest_tiles.txt 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_tiles.txt
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
source tools/ncu_cap.sh
export TRACE_REPS=1
cap flat_c$C $C auto node_prune_flat 5
cap cands_c$C $C auto tile_cands_kernel 5
cap k1t_c$C $C auto assign_tiles 5
for n in flat_c$C cands_c$C k1t_c$C; do
  zcat $O/ncu_${n}_source.csv.gz > /tmp/src.csv; python tools/ncu_lines.py /tmp/src.csv 45 > $O/ncu_${n}_lines.txt 2>&1
done
