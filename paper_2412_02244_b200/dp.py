"""Data-parallel Lloyd over shards (NEXT-3; the paper lists distribution as future work).

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch), points sharded, every
rank holding all k centroids.  Per iteration each rank runs the local assignment +
fixed-point accumulation (km_dp_step), ONE all-reduce sums the partial (k*(d+1)+2 int64
words: sums, counts, changed_t, SSE_t; 32 KB at k = 1000, d = 3), and every rank applies the
identical refine (km_dp_apply).  The sums are exact integers, so the result is bit-identical
to a single GPU holding all points, the final Eq. 1 included (128-bit fixed point, summed as
three 48-bit limbs).  This module is host orchestration only; every step of the path
runs in libkm (km_dp_* in include/km.h).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import km as _km


class LibkmShard:
    """This rank's shard on its GPU: a km_ctx and the device buffers of the partials."""

    def __init__(self, points, k: int, mode: int = _km.KM_MODE_AUTO, stream=None):
        import torch
        self.torch = torch
        self.points = points
        self.n, self.d = points.shape
        self.k = k
        self.ctx = _km.Context(self.n, self.d, k, stream)
        _km.km_set_mode(self.ctx.handle, mode)
        dev = points.device
        # sums [k][d], counts [k], changed; the high-d variant appends its moment sums Q [k]
        # (and its sums run over the padded width): the library gives the length
        self.partial = torch.zeros(_km.km_dp_partial_len(self.ctx.handle), dtype=torch.int64, device=dev)

    def bbox(self) -> np.ndarray:
        return _km.km_dp_bbox(self.ctx.handle, self.points)

    def begin(self, init, lo_hi, n_global: int, max_iter: int) -> None:
        _km.km_dp_begin(self.ctx.handle, self.points, init, lo_hi, n_global, max_iter)

    def step(self):
        _km.km_dp_step(self.ctx.handle, self.partial)
        return self.partial

    def apply(self, partial, tol: float, want_done: bool):
        return _km.km_dp_apply(self.ctx.handle, partial, tol, want_done)

    def end(self):
        """(centroids, this shard's labels, iterations, Eq. 1 of the shard as 3 int64 limbs)"""
        C = self.torch.empty((self.k, self.d), dtype=self.torch.float32, device=self.points.device)
        lab = self.torch.empty(self.n, dtype=self.torch.int32, device=self.points.device)
        it, _, limbs = _km.km_dp_end(self.ctx.handle, C, lab)
        return C, lab, it, limbs

    def sse(self, limbs_sum) -> float:
        return _km.km_dp_sse(self.ctx.handle, limbs_sum)

    def close(self):
        self.ctx.close()


@dataclass
class DPResult:
    centroids: object      # [k][d] float32 (identical on every rank)
    labels: object         # this rank's [n_local] int32
    sse: float             # Eq. 1 over ALL ranks
    iterations: int


def _allreduce(t, op, group):
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=op, group=group)
    return t


def lloyd_dp(shard, init, max_iter: int, tol: float = -1.0, group=None, comm_device=None) -> DPResult:
    """The data-parallel loop.  `shard` is a LibkmShard (or any object with the same
    methods); collectives run on `comm_device` tensors (cuda for NCCL, cpu for gloo)."""
    import torch
    import torch.distributed as dist
    R = dist.ReduceOp
    d = shard.d
    dev = comm_device if comm_device is not None else getattr(shard.points, "device", "cpu")
    lo_hi = shard.bbox()
    lo = torch.from_numpy(np.ascontiguousarray(lo_hi[:d])).to(dev)
    hi = torch.from_numpy(np.ascontiguousarray(lo_hi[d:])).to(dev)
    nt = torch.tensor([shard.n], dtype=torch.int64, device=dev)
    _allreduce(lo, R.MIN, group)
    _allreduce(hi, R.MAX, group)
    _allreduce(nt, R.SUM, group)
    glob = np.concatenate([lo.cpu().numpy(), hi.cpu().numpy()]).astype(np.float32)
    shard.begin(init, glob, int(nt.item()), max_iter)
    for _ in range(max_iter):
        part = shard.step()
        _allreduce(part, R.SUM, group)     # the one exchange: int64 sums, counts, changed_t, SSE_t
        _, done = shard.apply(part, tol, tol >= 0)
        if done:
            break
    C, lab, it, limbs = shard.end()
    lt = torch.from_numpy(np.asarray(limbs, np.int64)).to(dev)
    _allreduce(lt, R.SUM, group)           # Eq. 1: 128-bit fixed point in 48-bit limbs
    return DPResult(C, lab, shard.sse(lt.cpu().numpy()), it)


def lloyd_multi_shard(shards, init, max_iter: int, tol: float = -1.0) -> list:
    """Several shards driven from ONE process (e.g. several GPUs of one node without
    torch.distributed, or shards of one GPU in tests): the all-reduce is an in-process
    sum of the shards' partials.  Returns one DPResult per shard."""
    import torch
    d = shards[0].d
    boxes = [s.bbox() for s in shards]
    glob = np.concatenate([np.min([b[:d] for b in boxes], 0), np.max([b[d:] for b in boxes], 0)]).astype(np.float32)
    n_global = sum(s.n for s in shards)
    for s in shards:
        s.begin(init, glob, n_global, max_iter)
    for _ in range(max_iter):
        parts = [s.step() for s in shards]
        dev0 = parts[0].device
        tot = sum(p.to(dev0) for p in parts)
        done = False
        for s in shards:
            _, dn = s.apply(tot.to(s.partial.device), tol, tol >= 0)
            done = done or bool(dn)
        if done:
            break
    outs = [s.end() for s in shards]
    limbs = np.sum([np.asarray(o[3], np.int64) for o in outs], axis=0)
    sse_tot = shards[0].sse(limbs)
    return [DPResult(C, lab, sse_tot, it) for (C, lab, it, _) in outs]


def bench_dp(args, world, rank, local, synth, metric, unit, extras=None):
    """bench.py --gpus N under torchrun.  Weak scaling (default): one config-sized shard per rank
    (an independent instance seeded by the rank; shared initial centroids).  --scaling strong:
    the config's own points split over the ranks (config 4: 1e7 / N per GPU).  One step = the
    config's full run over all ranks' points; device time = the max over ranks.  `extras`
    (from bench.py) supplies the clock sampler and the roofline of the dominant kernel."""
    import json
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    strong = getattr(args, "scaling", "weak") == "strong"
    w0 = synth.config(args.config)                 # shared initial centroids (seed 0)
    if strong:
        # strong scaling: the config's points split into `world` contiguous shards
        idx = np.array_split(np.arange(w0.n), world)[rank]
        wr = synth.Workload(w0.name, np.ascontiguousarray(w0.points[idx]), w0.init, w0.iters, w0.desc)
    else:
        wr = synth.config(args.config, seed=rank)  # weak scaling: this rank's shard is an independent instance
    n, d, k = wr.n, wr.d, wr.k
    n_total = w0.n if strong else world * n
    P = torch.from_numpy(wr.points).to(dev)
    C0 = torch.from_numpy(w0.init).to(dev)
    mode = {"auto": _km.KM_MODE_AUTO, "brute": _km.KM_MODE_BRUTE, "tiles": _km.KM_MODE_TILES}[args.mode]
    stream = torch.cuda.current_stream(dev)
    shard = LibkmShard(P, k, mode, stream.cuda_stream)
    K, W = args.steps, max(args.warmup, 3)
    T = wr.iters

    def timed(steps, host=False, instrument=False, sampler=None):
        Ph = torch.from_numpy(wr.points).pin_memory() if host else None
        Lh = torch.empty(n, dtype=torch.int32).pin_memory() if host else None
        Ch = torch.empty((k, d), dtype=torch.float32).pin_memory() if host else None
        _km.km_timing_enable(shard.ctx.handle, instrument)
        _km.km_timing_read(shard.ctx.handle, reset=True)
        _km.km_launch_count(shard.ctx.handle, reset=True)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        if sampler is not None:
            sampler.__enter__()
        e0.record(stream)
        for _ in range(steps):   # one step = the config's full run (T iterations), as in the 1-GPU bench
            if host:
                P.copy_(Ph, non_blocking=True)                  # this step's points, pinned host -> device
            res = lloyd_dp(shard, C0, T, -1.0)
            assert res.iterations == T
            if host:
                Lh.copy_(res.labels)                             # the step's labels back to the host
                Ch.copy_(res.centroids)
        e1.record(stream)
        torch.cuda.synchronize()
        if sampler is not None:
            sampler.__exit__()
        dist.barrier()
        ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        launches = _km.km_launch_count(shard.ctx.handle)
        tm = _km.km_timing_read(shard.ctx.handle, reset=True)
        _km.km_timing_enable(shard.ctx.handle, False)
        return float(ms.item()), res, launches, tm

    for _ in range(W):
        lloyd_dp(shard, C0, T, -1.0)
    sampler = extras["sampler"](local) if extras else None
    ms_total, res, launches, _ = timed(K, sampler=sampler)
    ms_e2e, _, _, _ = timed(K, host=True)
    Ki = max(1, min(K, 3))
    ms_i, _, _, tm = timed(Ki, instrument=True)
    st = _km.km_read_stats(shard.ctx.handle)
    if rank == 0:
        ms_step = ms_total / K
        value = n_total * k * T / (ms_step * 1e-3)
        line = {"metric": metric, "value": value, "unit": unit, "n_gpus": world,
                "steps": K, "warmup": W, "ms_per_step": ms_step, "ms_per_iter": ms_step / T,
                "higher_is_better": True, "scaling": "strong" if strong else "weak",
                "vs_baseline": None,
                "dtype": ("tf32x3 tensor scores / f64 certify / int64 sums" if d > 3 else
                          "f32 scan / f64 certify / int64 sums"), "data": "synthetic",
                "config": {"workload": wr.name, "n_total": n_total, "n_per_rank": n, "d": d, "k": k, "mode": args.mode,
                           "iterations_per_step": T,
                           "parallelism": f"dp{world} (points sharded, one int64 all-reduce of k*(d+1)+2 "
                                          "words per iteration over NCCL: sums, counts, changed_t, SSE_t)",
                           "step": f"the config's full run ({T} Lloyd iterations) over all ranks' points"},
                "gpu_launches": launches,
                "e2e": {"value": n_total * k * T / (ms_e2e / K * 1e-3), "unit": unit, "ms_per_step": ms_e2e / K,
                        "h2d_bytes_per_step": n * d * 4, "d2h_bytes_per_step": n * 4 + k * d * 4,
                        "note": "per rank: the shard's points from pinned host memory, labels and centroids back, "
                                "every step (bytes per rank)"},
                "clocks": sampler.summary() if sampler is not None else None,
                "sse": res.sse}
        if extras:
            line["roofline"] = extras["roofline"](wr, {"timing": tm, "stats": st, "changed_t": [0] * T,
                                                       "ms_total": ms_i}, Ki)
        print(json.dumps(line), flush=True)
    shard.close()
    dist.destroy_process_group()
    return 0
