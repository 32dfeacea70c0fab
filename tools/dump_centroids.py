"""Centroids after every iteration of a config run (analysis of per-centroid drift):
python tools/dump_centroids.py <config> <out.npz>"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_2412_02244_b200 as kmb
cfg = int(sys.argv[1]); out = sys.argv[2]
w = synth.config(cfg)
P = torch.from_numpy(w.points).cuda(); C0 = torch.from_numpy(w.init).cuda()
C = torch.empty_like(C0); L = torch.empty(w.n, dtype=torch.int32, device="cuda")
ctx = kmb.Context(w.n, w.d, w.k)
cs = [w.init.copy()]
for t in range(1, w.iters + 1):
    kmb.km_run_ctx(ctx.handle, P, C0, t, -1.0, C, L)
    cs.append(C.cpu().numpy().copy())
np.savez_compressed(out, C=np.stack(cs))
ctx.close()
