#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tiles.py -x -q > gpurun_out/pytest_tiles.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_tiles.txt
for lib in default late; do
  if [ $lib = default ]; then L=$PWD/paper_2412_02244_b200/libkm.so; else L=$PWD/build/var/libkm_$lib.so; fi
  for c in 4 5 3; do KM_LIB_PATH=$L timeout 300 python bench.py --config $c --steps 200 --warmup 3 --no-cpu-baseline --no-brute > gpurun_out/tl_${lib}_c$c.json 2>/dev/null; done
done
for c in 4 5; do KM_LIB_PATH=$PWD/build/var/libkm_prof.so python tools/prof_tiles.py $c > gpurun_out/prof_sections_c$c.txt 2>&1; KM_LIB_PATH=$PWD/build/var/libkm_lateprof.so python tools/prof_tiles.py $c > gpurun_out/prof_sections_late_c$c.txt 2>&1; done
