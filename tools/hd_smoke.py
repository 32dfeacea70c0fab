"""Quick check of the high-dimensional path: one iteration vs the oracle (tools only)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
import paper_2412_02244_b200 as kmb
from paper_2412_02244_b200 import km as kmlib
for (n, d, k) in [(1000, 128, 37), (3001, 256, 300), (130, 32, 7)]:
    P, C0 = synth.random_instance(1, n, d, k, "blobs")
    ctx = kmb.Context(n, d, k)
    Cout = torch.empty((k, d), dtype=torch.float32, device="cuda"); lab = torch.empty(n, dtype=torch.int32, device="cuda")
    it, sse = kmb.km_run_ctx(ctx.handle, torch.from_numpy(P).cuda(), torch.from_numpy(C0).cuda(), 1, -1.0, Cout, lab)
    st = kmlib.km_hd_stats(ctx.handle)
    a = oracle.assign(P, C0.astype(np.float64))
    L = lab.cpu().numpy()
    print(n, d, k, "it", it, "mismatch", int((L != a.labels).sum()), "stats", st, "sse", sse, flush=True)
    ctx.close()
