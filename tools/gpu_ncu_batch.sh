#!/bin/bash
# Several ncu --set full captures (one kernel each) + centroid dumps:  tools/gpu_ncu_batch.sh TAG [caps...]
# Each report is exported (details text, raw csv, source csv) and deleted on the box (gpurun_out <= 64 MiB).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/$1
O=gpurun_out/$1
export TRACE_REPS=1
[ -n "$DUMP" ] && for c in 4 5; do timeout 300 python tools/dump_centroids.py $c $O/centroids_c$c.npz; echo "dump c$c rc=$?"; done
cap() {  # name config mode regex skip
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$4 -s $5 -c 1 \
    -o $O/ncu_$1 python tools/trace_run.py $2 $3 > $O/ncu_$1.log 2>&1; echo "ncu $1 rc=$?"
  ncu -i $O/ncu_$1.ncu-rep --page details > $O/ncu_$1_details.txt 2>&1
  ncu -i $O/ncu_$1.ncu-rep --page raw --csv > $O/ncu_$1_raw.csv 2>&1
  ncu -i $O/ncu_$1.ncu-rep --page source --csv > $O/ncu_$1_source.csv 2>&1
  gzip -f $O/ncu_$1_source.csv $O/ncu_$1_raw.csv
  if [ $(stat -c %s $O/ncu_$1.ncu-rep) -gt 6000000 ]; then rm -f $O/ncu_$1.ncu-rep; fi
}
cap c4_nodeflat 4 auto node_prune_flat 5
cap c4_tcands 4 auto tile_cands_kernel 5
cap c4_k1t 4 auto assign_tiles 5
cap c2_k1 2 auto assign_scan 5
cap c1_small 1 auto lloyd_small 2
cap c4_geom 4 auto tile_geom 0
cap c4_scatter 4 auto scatter_labels 0
du -sh $O
