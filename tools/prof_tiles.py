"""Section-cycle profile of the tile kernel (KM_PROF build): python tools/prof_tiles.py <config>"""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_2412_02244_b200 as kmb
from paper_2412_02244_b200 import km as kmlib
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
w = synth.config(cfg)
P = torch.from_numpy(w.points).cuda(); C0 = torch.from_numpy(w.init).cuda()
C = torch.empty_like(C0); L = torch.empty(w.n, dtype=torch.int32, device="cuda")
ctx = kmb.Context(w.n, w.d, w.k)
kmb.km_set_mode(ctx.handle, kmb.KM_MODE_TILES)
kmb.km_run_ctx(ctx.handle, P, C0, 5, -1.0, C, L)
iters = 10
kmb.km_run_ctx(ctx.handle, P, C0, iters, -1.0, C, L)
f = kmlib._lib.km_debug_stats
f.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
out = np.zeros(32, np.int64)
f(ctx.handle, out.ctypes.data)
names = ["pairs", "pts", "batch", "tiles", "wait", "list_stage", "batch_path", "scan", "certify", "accum", "sum_plen", "list_in_smem", "eq5_tiles", "eq4_tiles", "pretest", "prune_core", "prune_smem", "prune_global", "n_global", "plen_global", "w_issue", "w_list", "eq4_points", "w_lane0", "t>20k", "t>50k", "t>200k", "tmax", "cyc_in_>50k"]
tiles = out[3]
for i, nm in enumerate(names):
    v = out[i]
    extra = f"  per tile {v / tiles:.1f}" if i >= 4 and i not in (12, 13, 18, 19, 22, 24, 25, 26, 27, 28) else ""
    print(f"{nm:14s} {v:16d}{extra}")
