#!/bin/bash
# round-end check: all GPU tests, smoke, default bench, high-d bench, reference arm, HD ncu
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-final}
timeout 1200 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/pytest_gpu_$TAG.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_$TAG.txt
tail -3 gpurun_out/pytest_gpu_$TAG.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$TAG.txt 2>&1; echo "rc=$?" >> gpurun_out/smoke_$TAG.txt
tail -2 gpurun_out/smoke_$TAG.txt
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 600 python bench.py --config 6 --steps 10 > gpurun_out/bench_c6_$TAG.json 2> gpurun_out/bench_c6_$TAG.err; echo "bench c6 rc=$?"
timeout 600 python bench.py --config 7 --steps 5 --cpu-seconds 10 > gpurun_out/bench_c7_$TAG.json 2> gpurun_out/bench_c7_$TAG.err; echo "bench c7 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c6_$TAG.csv python tools/hd_bench.py 6 1000 3 > /dev/null 2>&1; echo "ncu launches rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:hd_gemm -s 2 -c 1 -o gpurun_out/hd_gemm_$TAG python tools/hd_bench.py 6 1000 2 > /dev/null 2>&1; echo "ncu full rc=$?"
