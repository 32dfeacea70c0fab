#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tiles.py -x -q > gpurun_out/pytest_tiles.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_tiles.txt
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_tiles.json 2> gpurun_out/bench_tiles.err
timeout 300 python bench.py --config 5 --steps 20 --warmup 3 --no-cpu-baseline --no-brute > gpurun_out/bench_tiles_c5.json 2> gpurun_out/bench_tiles_c5.err
timeout 300 python bench.py --config 3 --steps 200 --warmup 3 --no-cpu-baseline > gpurun_out/bench_tiles_c3.json 2> gpurun_out/bench_tiles_c3.err
timeout 300 python bench.py --config 2 --steps 200 --warmup 3 --no-cpu-baseline > gpurun_out/bench_tiles_c2.json 2> gpurun_out/bench_tiles_c2.err
