cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
export TRACE_REPS=1
for dbg in "" "6=1" "6=2"; do
  tag=L${dbg//=/_}
  KM_TRACE_DBG=$dbg timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
    python tools/trace_run.py ${CFG:-4} > gpurun_out/trace_$tag.json 2>&1; echo "launches $tag rc=$?"
  python tools/launch_summary.py gpurun_out/launches_$tag.csv > gpurun_out/launches_${tag}_summary.txt 2>&1
  grep -E "cand|prune|tile_cands|assign_tiles<3, 0|launches" gpurun_out/launches_${tag}_summary.txt
done
