"""One high-dimensional run (tools only): python tools/hd_one.py n d k iters [kind]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
import paper_2412_02244_b200 as kmb
from paper_2412_02244_b200 import km as kmlib
n, d, k, it = map(int, sys.argv[1:5]); kind = sys.argv[5] if len(sys.argv) > 5 else "blobs"
P, C0 = synth.random_instance(7 * n + d + k, n, d, k, kind)
ctx = kmb.Context(n, d, k)
Cout = torch.empty((k, d), dtype=torch.float32, device="cuda"); lab = torch.empty(n, dtype=torch.int32, device="cuda")
r, sse = kmb.km_run_ctx(ctx.handle, torch.from_numpy(P).cuda(), torch.from_numpy(C0).cuda(), it, -1.0, Cout, lab)
st = kmlib.km_hd_stats(ctx.handle)
a = oracle.assign(P, C0.astype(np.float64)) if it == 1 else None
mm = int((lab.cpu().numpy() != a.labels).sum()) if a is not None else -1
print(n, d, k, it, kind, "iters", r, "stats", st, "mismatch", mm, flush=True)
