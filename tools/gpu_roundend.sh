#!/bin/bash
# Checkpoint run: GPU suite, smoke, bench lines for configs 1-7, reference arm, config-4 launch
# list and one ncu --set full capture of K1t.   tools/gpu_roundend.sh TAG
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/$1
O=gpurun_out/$1
timeout 1500 python -m pytest tests -m gpu -x -q --durations=8 > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
tail -2 $O/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
for c in 1 2 3 5; do
  timeout 900 python bench.py --config $c --steps 10 > $O/bench_config$c.json 2> $O/bench_config$c.err; echo "bench c$c rc=$?"
done
for c in 6 7; do
  timeout 900 python bench.py --config $c --steps 5 --cpu-seconds 10 > $O/bench_config$c.json 2> $O/bench_config$c.err; echo "bench c$c rc=$?"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?"
export TRACE_REPS=1
timeout 300 python tools/trace_run.py 4 > $O/trace_c4.json 2> $O/trace_c4.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv \
    python tools/trace_run.py 4 > /dev/null 2>&1; echo "launches rc=$?"
python tools/launch_summary.py $O/launches_c4.csv > $O/launches_c4_summary.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:assign_tiles -s 5 -c 1 \
    -o $O/ncu_k1t_c4 python tools/trace_run.py 4 > $O/ncu_k1t.log 2>&1; echo "ncu rc=$?"
