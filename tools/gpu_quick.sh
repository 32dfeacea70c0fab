#!/bin/bash
# Quick check: tile-path GPU tests + bench lines for configs 4 (default), 3, 2, 5 + launch list of config 4.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-q}
timeout 900 python -m pytest tests/test_gpu_tiles.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_quick_$TAG.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick_$TAG.txt
tail -3 gpurun_out/pytest_quick_$TAG.txt
for c in 4 3 2 5; do
  timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline --no-brute > gpurun_out/bench_${TAG}_c$c.json 2> gpurun_out/bench_${TAG}_c$c.err; echo "bench c$c rc=$?"
done
export TRACE_REPS=1
for c in ${LCFGS:-4}; do
timeout 300 python tools/trace_run.py $c > gpurun_out/trace_${TAG}_c$c.json 2> gpurun_out/trace_${TAG}_c$c.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control ${NCU_CACHE:-all} --csv --log-file gpurun_out/launches_${TAG}_c$c.csv \
    python tools/trace_run.py $c > /dev/null 2>&1; echo "launches c$c rc=$?"
python tools/launch_summary.py gpurun_out/launches_${TAG}_c$c.csv > gpurun_out/launches_${TAG}_c${c}_summary.txt 2>&1
done
