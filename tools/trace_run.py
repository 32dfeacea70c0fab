"""Per-iteration picture of one config run: traces (SSE_t, changed_t, max drift), the tile
path's work counters and per-kernel device times.  python tools/trace_run.py <config> [mode]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_2412_02244_b200 as kmb
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
mode = {"tiles": kmb.KM_MODE_TILES, "brute": kmb.KM_MODE_BRUTE, "auto": kmb.KM_MODE_AUTO}[sys.argv[2] if len(sys.argv) > 2 else "auto"]
w = synth.config(cfg)
P = torch.from_numpy(w.points).cuda(); C0 = torch.from_numpy(w.init).cuda()
C = torch.empty_like(C0); L = torch.empty(w.n, dtype=torch.int32, device="cuda")
ctx = kmb.Context(w.n, w.d, w.k)
kmb.km_set_mode(ctx.handle, mode)
for kv in filter(None, os.environ.get("KM_TRACE_DBG", "").split(",")):   # e.g. KM_TRACE_DBG=6=1,1=4
    kk, vv = kv.split("=")
    kmb.km.km_debug_set(ctx.handle, int(kk), int(vv))
for _ in range(2):
    kmb.km_run_ctx(ctx.handle, P, C0, w.iters, -1.0, C, L)
torch.cuda.synchronize()
times = []
for _ in range(int(os.environ.get("TRACE_REPS", "7"))):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); it, sse = kmb.km_run_ctx(ctx.handle, P, C0, w.iters, -1.0, C, L); e1.record(); torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
ms = sorted(times)[len(times) // 2]   # median of the repetitions
tr = kmb.km_read_traces(ctx.handle, w.iters)
st = kmb.km_read_stats(ctx.handle)
kmb.km_timing_enable(ctx.handle, True); kmb.km_timing_read(ctx.handle, reset=True)
kmb.km_run_ctx(ctx.handle, P, C0, w.iters, -1.0, C, L); torch.cuda.synchronize()
tm = kmb.km_timing_read(ctx.handle, reset=True)
print(json.dumps({"config": cfg, "iters": it, "ms_run": ms, "ms_per_iter": ms / w.iters, "sse": sse, "stats": st,
                  "timing": tm, "sse_t": list(map(float, tr.sse)), "changed_t": list(map(int, tr.changed)),
                  "max_drift_t": list(map(float, tr.max_drift))}))
ctx.close()
