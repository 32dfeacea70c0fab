#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dp.py -x -q > gpurun_out/pytest_dp.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_dp.txt
# single-GPU torchrun smoke of the NCCL path (world size 1)
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 1 --steps 20 --warmup 3 > gpurun_out/bench_dp1.json 2> gpurun_out/bench_dp1.err; echo "rc=$?" >> gpurun_out/bench_dp1.err
