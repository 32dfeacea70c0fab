#!/bin/bash
# quick timing of the high-dimensional configs (tools only)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for c in "6 1000" "7 1000" "6 10000" "7 10000"; do
  timeout 90 python tools/hd_bench.py $c > gpurun_out/hb_$(echo $c | tr ' ' _).json 2>&1
  python3 -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(d['config'], d['k'], round(d['ms_per_iter'],3), d['stats'])" gpurun_out/hb_$(echo $c | tr ' ' _).json
done
