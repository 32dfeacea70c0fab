#!/bin/bash
# session 2: probe, variant benches, tests, then ncu (launch list + full capture of the assign kernel)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 120 ./build/fp32_probe > gpurun_out/probe2.txt 2>&1
for v in 1 2; do
  timeout 300 python bench.py --steps 100 --warmup 10 --variant $v --no-cpu-baseline > gpurun_out/bench_v$v.json 2> gpurun_out/bench_v$v.err
done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu2.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu2.txt
CMD="python bench.py --steps 3 --warmup 3 --variant 2 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:assign_chunk -s 2 -c 1 -o gpurun_out/prof_chunk $CMD > gpurun_out/ncu_full.log 2>&1
echo done
