#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
cat > /tmp/mc.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, synth
import paper_2412_02244_b200 as kmb
w = synth.config(1, n=50000, k=10)
P = torch.from_numpy(w.points).cuda(); C0 = torch.from_numpy(w.init).cuda()
C = torch.empty_like(C0); L = torch.empty(w.n, dtype=torch.int32, device="cuda")
ctx = kmb.Context(w.n, w.d, w.k); kmb.km_set_mode(ctx.handle, kmb.KM_MODE_TILES)
print(kmb.km_run_ctx(ctx.handle, P, C0, 3, -1.0, C, L))
PY
timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python /tmp/mc.py > gpurun_out/memcheck.txt 2>&1
echo "rc=$?" >> gpurun_out/memcheck.txt
