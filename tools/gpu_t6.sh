cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
export TRACE_REPS=1
for m in auto brute; do
timeout 900 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_elapsed.avg --clock-control none --csv --log-file gpurun_out/l6_$m.csv \
    python tools/trace_run.py 2 $m > gpurun_out/trace6_$m.json 2>&1; echo "launches rc=$?"
python tools/launch_summary.py gpurun_out/l6_$m.csv > gpurun_out/l6_${m}_summary.txt 2>&1
cat gpurun_out/l6_${m}_summary.txt
done
python - <<'P'
import csv
for m in ("auto","brute"):
    rows=[r for r in csv.reader(open(f"gpurun_out/l6_{m}.csv")) if len(r)>10]
    h=rows[0]; iN=h.index("Kernel Name"); iM=h.index("Metric Name"); iV=h.index("Metric Value")
    out=[(r[iN][:30], r[iM], r[iV]) for r in rows[1:] if "scan" in r[iN]]
    for o in out[-9:]: print(m, o)
P
