"""High-dimensional variant timing (tools only): python tools/hd_bench.py CFG [k] [iters]"""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_2412_02244_b200 as kmb
from paper_2412_02244_b200 import km as kmlib
cfg = int(sys.argv[1]); k = int(sys.argv[2]) if len(sys.argv) > 2 else None
w = synth.config(cfg, k=k)
iters = int(sys.argv[3]) if len(sys.argv) > 3 else w.iters
P = torch.from_numpy(w.points).cuda(); C0 = torch.from_numpy(w.init).cuda()
C = torch.empty_like(C0); L = torch.empty(w.n, dtype=torch.int32, device="cuda")
ctx = kmb.Context(w.n, w.d, w.k)
for _ in range(2):
    kmb.km_run_ctx(ctx.handle, P, C0, iters, -1.0, C, L)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); kmb.km_run_ctx(ctx.handle, P, C0, iters, -1.0, C, L); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = sorted(ts)[2]
st = kmlib.km_hd_stats(ctx.handle)
kmb.km_timing_enable(ctx.handle, True); kmb.km_timing_read(ctx.handle, reset=True)
kmb.km_run_ctx(ctx.handle, P, C0, iters, -1.0, C, L); torch.cuda.synchronize()
tm = kmb.km_timing_read(ctx.handle, reset=True)
tr = kmb.km_read_traces(ctx.handle, iters)
flop = 2.0 * w.n * w.k * w.d * iters
print(json.dumps({"config": cfg, "n": w.n, "d": w.d, "k": w.k, "iters": iters, "ms_run": ms, "ms_per_iter": ms / iters,
                  "gemm_tflops_equiv": flop / (ms * 1e-3) / 1e12, "stats": st, "timing": tm,
                  "changed": list(map(int, tr.changed))}))
ctx.close()
