#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tiles.py tests/test_gpu_parity.py tests/test_gpu_dp.py -q -m gpu -x > gpurun_out/st_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/st_pytest.txt
O=gpurun_out/st_bench.txt; : > $O
for c in 4 3 5 2; do
  r=$(timeout 200 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-brute 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.readline()); print(d["ms_per_step"])')
  echo "c$c $r" >> $O
done
