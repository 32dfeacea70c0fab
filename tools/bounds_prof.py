"""Phase times of the bounds kernel (a -DKM_BPROF build): python tools/bounds_prof.py <config>"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2412_02244_b200 as kmb
from paper_2412_02244_b200 import km as kmlib
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = synth.config(cfg)
P = torch.from_numpy(w.points).cuda(); C0 = torch.from_numpy(w.init).cuda()
C = torch.empty_like(C0); L = torch.empty(w.n, dtype=torch.int32, device="cuda")
ctx = kmb.Context(w.n, w.d, w.k)
kmb.km_set_mode(ctx.handle, kmb.KM_MODE_BOUNDS)
for _ in range(3):
    kmb.km_run_ctx(ctx.handle, P, C0, w.iters, -1.0, C, L)
b = kmlib.km_debug_bounds(ctx.handle)
grid = kmlib._lib.km_debug_assign_grid(ctx.handle)
names = ["refine", "s_a pass", "bound test", "queued scan", "flush+partials"]
tot = sum(b[1:6])
print("points scanned", b[0])
for i, nm in enumerate(names):
    print(f"{nm:16s} {b[1 + i] / 1e3:10.1f} us summed over CTAs x iterations  {100 * b[1 + i] / max(tot, 1):5.1f} %")
ctx.close()
