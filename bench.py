#!/usr/bin/env python3
"""bench.py -- exact Lloyd step on one B200 (BASELINE.json headline: config 4,
n=1e7 d=3 k=1000), printed as ONE JSON line.

A "step" is the config's whole run as a user makes it: one km_run_ctx call of the
config's iteration count (20 at config 4; tol = -1, fixed count), including the
once-per-call index build, the final SSE and the labels in input order.  Lloyd
iterations are not interchangeable under pruning (late ones are cheaper), so the
step is the full run, not one iteration of a long run.  `--steps K` timed steps,
`--warmup W` untimed ones first.

value  = point-centroid distances/s = n*k*iters*K / device time (CUDA events on
         the library's stream), inputs already resident in HBM.
e2e    = same metric through km_run_ctx with PINNED HOST buffers (H2D of points
         and C0, D2H of labels, centroids and SSE inside every step).
roofline: the assignment kernel (dominant).  Brute force: FP32 CUDA-core bound
         ("alu"), 3*d*n*k FLOP per launch.  Tile path: the bytes of the tiles it
         must read against the measured HBM bandwidth.
         High-dimensional configs 6/7 (NEXT-4): the tcgen05 score kernel, "tensor"
         bound, 2*n*k*d FLOP per launch against the TF32 peak.
cpu_baseline: the FP64 oracle, as it stands, on a bounded sample, host cores.
--impl reference: the oracle as the reference arm (rank 0 only).
"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "k-means ms/iter and point-centroid distances/s at n=1e7 d=3 k=1000; % roofline"
UNIT = "distances/s"
SM_COUNT_NOMINAL = 148
FP32_LANES_PER_SM = 128
SM_MAX_MHZ_NOMINAL = 1965.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--variant", type=int, default=None, help="assign kernel variant (debug)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-brute", action="store_true", help="skip the brute-force comparison run")
    ap.add_argument("--mode", default="auto", choices=["auto", "brute", "tiles", "bounds"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="oracle sample budget")
    ap.add_argument("--dbg", type=lambda x: tuple(map(int, x.split("="))), action="append", default=[],
                    help="(tuning) km_debug_set KEY=VALUE, repeatable")
    ap.add_argument("--st-shift", type=int, default=None, help="(tuning) tiles per level-1 node = 2^value")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="--gpus N: a config-sized shard per rank (weak) or the config split over the ranks (strong)")
    return ap.parse_args()


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """NVML sampling of SM clock / throttle reasons during the timed region."""

    def __init__(self, index=0, period=0.005):
        self.samples, self.reasons, self.period = [], set(), period
        self.stop_evt = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = str(e)
            self.max_mhz = None

    _REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
                0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle"}

    def _run(self):
        while not self.stop_evt.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self._REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self.stop_evt.set()
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": getattr(self, "err", "no nvml")}
        load = [s for s in self.samples if s > 0]
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def cpu_baseline(w, seconds_budget, steps_hint=1):
    """Time the oracle, as it stands, on a bounded sample of the workload."""
    import oracle
    threads = oracle.max_threads()
    k = w.k
    # calibrate on a small sample, then size the sample to the budget
    n0 = min(w.n, max(2000, 2_000_000 // k))
    t0 = time.perf_counter()
    oracle.lloyd(w.points[:n0], w.init.astype(np.float64), 1, -1.0, True, threads=threads)
    dt0 = max(time.perf_counter() - t0, 1e-4)
    rate = n0 * k / dt0
    n_s = int(min(w.n, max(n0, seconds_budget * rate / k)))
    t0 = time.perf_counter()
    r = oracle.lloyd(w.points[:n_s], w.init.astype(np.float64), 1, -1.0, True, threads=threads)
    dt = time.perf_counter() - t0
    return {"value": n_s * k / dt, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"first {n_s} of {w.n} points of {w.name}, all k={k} centroids, 1 Lloyd iteration "
                      f"(FP64 oracle, OpenMP over points), {dt:.2f} s", "ms_per_iter_at_sample": dt * 1e3,
            "iterations": r.iterations}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    w = synth.config(args.config)
    threads = oracle.max_threads()
    k = w.k
    K, W = args.steps, max(args.warmup, 0)
    # each step: one oracle Lloyd iteration over a bounded sample (whole run ~ a few minutes)
    n0 = min(w.n, max(2000, 2_000_000 // k))
    t0 = time.perf_counter()
    oracle.lloyd(w.points[:n0], w.init.astype(np.float64), 1, -1.0, True, threads=threads)
    rate = n0 * k / max(time.perf_counter() - t0, 1e-4)
    budget = 150.0
    n_s = int(min(w.n, max(n0, budget * rate / (k * (K + W)))))
    sample = w.points[:n_s]
    C = w.init.astype(np.float64)
    for _ in range(W):
        oracle.lloyd(sample, C, 1, -1.0, True, threads=threads)
    t0 = time.perf_counter()
    for _ in range(K):
        oracle.lloyd(sample, C, 1, -1.0, True, threads=threads)
    dt = time.perf_counter() - t0
    ms = dt / K * 1e3
    val = n_s * k / (ms * 1e-3)
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": K,
            "warmup": W, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.name, "desc": w.desc, "n": w.n, "d": w.d, "k": w.k, "sample_n": n_s},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": f"first {n_s} points of {w.name}, all k={k}; each step = 1 FP64 Lloyd "
                                       f"iteration over the sample"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def traffic_from_profiles(workload):
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        return t.get(workload)
    except Exception:
        return None


def _peak_fp32(nsm, mhz=SM_MAX_MHZ_NOMINAL):
    return nsm * FP32_LANES_PER_SM * 2 * mhz * 1e6 / 1e12


def measured_fp32_peak():
    """The FFMA/FFMA2 microbenchmark (tools/fp32_probe.cu, run on a B200 of this pool; the
    best packed rate) in TFLOP/s (2 FLOP per lane-op), or None."""
    try:
        best = 0.0
        for line in open(os.path.join(ROOT, "profiles", "r01", "fp32_probe.jsonl")):
            r = json.loads(line)
            if str(r.get("probe", "")).startswith(("ffma", "fadd")):
                best = max(best, r["lane_ops_per_s"])
        return 2 * best / 1e12 if best else None
    except Exception:
        return None


def measure(kmb, kmlib, torch, w, dev, stream, mode, K, W, variant=None, sampler=None, instrument=False,
            host=False, st_shift=None, dbg=()):
    """W untimed warm-up runs, then EXACTLY K timed runs of the config (one step = one
    km_run_ctx call of w.iters Lloyd iterations, tol = -1: index build, iterations, final SSE,
    labels back in input order).  host=True: pinned host buffers (H2D / D2H inside every
    step).  instrument=True: CUDA events around every libkm launch (per-kernel times)."""
    n, d, k = w.n, w.d, w.k
    if host:
        Pd = torch.from_numpy(w.points).pin_memory()
        C0d = torch.from_numpy(w.init).pin_memory()
        Cout = torch.empty((k, d), dtype=torch.float32).pin_memory()
        lab = torch.empty(n, dtype=torch.int32).pin_memory()
    else:
        Pd = torch.from_numpy(w.points).to(dev)
        C0d = torch.from_numpy(w.init).to(dev)
        Cout = torch.empty((k, d), dtype=torch.float32, device=dev)
        lab = torch.empty(n, dtype=torch.int32, device=dev)
    ctx = kmb.Context(n, d, k, stream.cuda_stream)
    kmb.km_set_mode(ctx.handle, mode)
    if variant is not None:
        kmlib.km_debug_set_variant(ctx.handle, variant)
    if st_shift is not None:
        kmlib.km_debug_set(ctx.handle, kmlib.KM_DBG_ST_SHIFT, st_shift)
    for key, val in dbg:
        kmlib.km_debug_set(ctx.handle, key, val)
    for _ in range(W):
        kmb.km_run_ctx(ctx.handle, Pd, C0d, w.iters, -1.0, Cout, lab)
    torch.cuda.synchronize()
    kmb.km_timing_enable(ctx.handle, instrument)
    kmb.km_timing_read(ctx.handle, reset=True)
    kmb.km_launch_count(ctx.handle, reset=True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if sampler is not None:
        sampler.__enter__()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
    ev0.record(stream)
    evs[0].record(stream)
    sses = []
    for i in range(K):
        it, sse = kmb.km_run_ctx(ctx.handle, Pd, C0d, w.iters, -1.0, Cout, lab)
        assert it == w.iters, (it, w.iters)
        sses.append(sse)
        evs[i + 1].record(stream)
    ev1.record(stream)
    torch.cuda.synchronize()
    per_step = [evs[i].elapsed_time(evs[i + 1]) for i in range(K)]
    if sampler is not None:
        sampler.__exit__()
    launches = kmb.km_launch_count(ctx.handle)
    tm = kmb.km_timing_read(ctx.handle, reset=True)
    st = kmb.km_read_stats(ctx.handle)   # counters of the last step
    tr = kmb.km_read_traces(ctx.handle, w.iters)
    kmb.km_timing_enable(ctx.handle, False)
    ctx.close()
    total_ms = ev0.elapsed_time(ev1)
    assert all(x == sses[0] for x in sses), "steps must be bit-identical"
    return {"ms_total": total_ms, "ms_per_step": total_ms / K, "ms_per_iter": total_ms / K / w.iters,
            "ms_per_step_median": statistics.median(per_step), "ms_per_step_min": min(per_step),
            "sse": sses[0], "launches": launches, "timing": tm, "stats": st, "changed_t": list(map(int, tr.changed))}


def tf32_peak():
    """Dense TF32 tensor peak: the measured bf16 cuBLAS number x the nominal TF32/BF16 ratio
    (1.1 / 2.25 PFLOP/s dense per GPU, B200_PROFILING.md)."""
    pk = peaks()
    bf16 = pk.get("bf16_tflops")
    if bf16:
        return bf16 * 0.5, "MEASURED_PEAKS.json bf16_tflops %.1f x 0.5 (nominal TF32/BF16 ratio)" % bf16
    return 1100.0, "nominal dense TF32 1.1 PFLOP/s (no measured peak)"


def kernel_roofline(w, r, K, nsm, hbm_gbs):
    """Roofline of the dominant kernel (the assignment) from an instrumented measurement."""
    n, d, k, T = w.n, w.d, w.k, w.iters
    tm, st = r["timing"], r["stats"]
    a_ms = tm["assign_ms"] / max(tm["assign_launches"], 1)
    peak = _peak_fp32(nsm)
    if d > 3:
        # high-dimensional variant: the score contraction p'.c' for all n x k pairs (2 d FLOP
        # each) on the tensor cores.  Split products: hi.hi in TF32 + two BF16 corrections (BF16
        # runs at twice the TF32 rate), i.e. tensor time of 2x these FLOPs at the TF32 rate
        flops = 2.0 * n * k * d
        tpk, note = tf32_peak()
        achieved = flops / (a_ms * 1e-3) / 1e12
        return {"bound": "tensor", "achieved": achieved, "peak": tpk, "unit": "TFLOP/s", "frac": achieved / tpk,
                "kernel": "hd_gemm_kernel (tcgen05.mma: TF32 hi.hi + 2 BF16 correction products)",
                "flop_per_launch": flops, "mma_flop_issued_per_launch": 3 * flops, "gemm_ms_per_launch": a_ms,
                "tensor_time_frac": 2 * achieved / tpk,
                "tensor_time_note": "TF32-equivalent MMA time issued (1 TF32 + 2 BF16 products per element) / peak",
                "peak_source": note}
    if not st["tiles"] and st["points_scanned"] < T * n:
        # KM_MODE_BOUNDS (bounds_scan_kernel): every point streams its coordinates, label and
        # bound (read) and its bound (write); the points that fail the bound test scan all k
        pairs = st["pairs"] / T
        flops = 3.0 * d * pairs
        bytes_ = n * (4 * d + 4 + 4 + 4) + sum(r["changed_t"]) / T * 4
        t_alu = flops / (peak * 1e12)
        t_hbm = bytes_ / (hbm_gbs * 1e9)
        t = a_ms * 1e-3
        common = {"kernel": "bounds_scan_kernel (K1b, brute force + per-point Hamerly bounds)",
                  "pairs_per_launch": pairs, "points_scanned_per_launch": st["points_scanned"] / T,
                  "bytes_per_launch": bytes_, "assign_ms_per_launch": a_ms, "hbm_time_ms": t_hbm * 1e3,
                  "alu_time_ms": t_alu * 1e3,
                  "bytes_note": "per point: coordinates, label, bound read + bound written; +4 B per changed label"}
        if t_alu >= t_hbm:
            return dict({"bound": "alu", "achieved": flops / t / 1e12, "peak": peak, "unit": "TFLOP/s",
                         "frac": t_alu / t}, **common)
        return dict({"bound": "hbm", "achieved": bytes_ / t / 1e9, "peak": hbm_gbs, "unit": "GB/s",
                     "frac": t_hbm / t}, **common)
    if not st["tiles"]:
        flops = 3.0 * d * n * k
        achieved = flops / (a_ms * 1e-3) / 1e12
        return {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "kernel": "assign_scan_kernel (K1, brute force)", "flop_per_pair": 3 * d,
                "pairs_per_launch": n * k, "assign_ms_per_launch": a_ms}
    # tile path (counters of one step = T launches): FLOPs of the pairs evaluated, bytes of the
    # tiles the kernel must read (points + previous labels + 96 B tile record) and label writes
    pairs = st["pairs"] / T
    visits = st["tile_visits"] / T
    flops = 3.0 * d * pairs
    bytes_ = visits * (128 * (4 * d + 4) + 96 + 16) + sum(r["changed_t"]) / T * 4
    t_alu = flops / (peak * 1e12)
    t_hbm = bytes_ / (hbm_gbs * 1e9)
    t = a_ms * 1e-3
    common = {"kernel": "assign_tiles_kernel (K1t, inter-bound + tile-pruned)", "pairs_per_launch": pairs,
              "tiles_per_launch": visits, "bytes_per_launch": bytes_, "assign_ms_per_launch": a_ms,
              "hbm_time_ms": t_hbm * 1e3, "alu_time_ms": t_alu * 1e3,
              "bytes_note": "per listed tile: 128 x (4d+4) B points + previous labels, 112 B tile record; "
                            "+4 B per changed label"}
    if t_alu >= t_hbm:
        return dict({"bound": "alu", "achieved": flops / t / 1e12, "peak": peak, "unit": "TFLOP/s",
                     "frac": t_alu / t}, **common)
    return dict({"bound": "hbm", "achieved": bytes_ / t / 1e9, "peak": hbm_gbs, "unit": "GB/s", "frac": t_hbm / t},
                **common)


def run_native(args):
    import torch
    import paper_2412_02244_b200 as kmb
    from paper_2412_02244_b200 import km as kmlib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or os.environ.get("KM_BENCH_FORCE_DP"):   # (the env: the DP path at one rank, for tests)
        return run_native_dp(args, world, rank, local)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    w = synth.config(args.config)
    n, d, k, T = w.n, w.d, w.k, w.iters
    K, W = args.steps, max(args.warmup, 3)
    stream = torch.cuda.current_stream(dev)
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    hbm = peaks().get("hbm_gbs", 6650.0)
    mode = {"auto": kmb.KM_MODE_AUTO, "brute": kmb.KM_MODE_BRUTE, "tiles": kmb.KM_MODE_TILES,
            "bounds": kmb.KM_MODE_BOUNDS}[args.mode]

    sampler = ClockSampler(local)
    r = measure(kmb, kmlib, torch, w, dev, stream, mode, K, W, args.variant, sampler, st_shift=args.st_shift, dbg=args.dbg)
    clocks = sampler.summary()
    value = n * k * T * K / (r["ms_total"] * 1e-3)
    # per-kernel device times from an instrumented measurement of the same steps
    ri = measure(kmb, kmlib, torch, w, dev, stream, mode, max(1, min(K, 5)), 1, args.variant, instrument=True,
                 st_shift=args.st_shift, dbg=args.dbg)
    Ki = max(1, min(K, 5))
    roof = kernel_roofline(w, ri, Ki, nsm, hbm)
    roof["traffic"] = traffic_from_profiles(w.name + ("_hd" if d > 3 else "_tiles" if r["stats"]["tiles"] else "_brute"))
    roof["peak_note"] = (f"alu: {nsm} SM x 128 FP32 lanes x 2 FLOP x 1965 MHz (guide unit counts, max clock); "
                         f"hbm: MEASURED_PEAKS.json hbm_gbs {hbm} (measured copy bandwidth); tensor: TF32 = "
                         f"measured bf16 x 0.5")
    hd_stats = None
    if d > 3:
        ctx = kmb.Context(n, d, k, stream.cuda_stream)
        Pd = torch.from_numpy(w.points).to(dev)
        C0d = torch.from_numpy(w.init).to(dev)
        Cout = torch.empty((k, d), dtype=torch.float32, device=dev)
        lab = torch.empty(n, dtype=torch.int32, device=dev)
        kmb.km_run_ctx(ctx.handle, Pd, C0d, T, -1.0, Cout, lab)
        hd_stats = kmlib.km_hd_stats(ctx.handle)
        ctx.close()
    tmi = ri["timing"]
    roof["assign_share_of_step"] = tmi["assign_ms"] / ri["ms_total"]
    breakdown = {"assign_ms_per_iter": tmi["assign_ms"] / (Ki * T), "finalize_ms_per_iter": tmi["update_ms"] / (Ki * T),
                 "other_ms_per_step": tmi["other_ms"] / Ki,
                 "other_note": "index build (bbox, Morton sort, gather, tile geometry) + per-iteration inter bound, "
                               "tile filter, prune of the index levels + final SSE and label scatter",
                 "instrumented_ms_per_step": ri["ms_per_step"]}

    # e2e: pinned host buffers through the same public call, H2D/D2H inside every step
    re = measure(kmb, kmlib, torch, w, dev, stream, mode, K, 1, args.variant, host=True, st_shift=args.st_shift, dbg=args.dbg)
    assert re["sse"] == r["sse"], (re["sse"], r["sse"])
    e2e_val = n * k * T * K / (re["ms_total"] * 1e-3)

    # the brute-force kernel beside it (context: the n x k scan the paper's method avoids)
    brute = None
    if r["stats"]["tiles"] and d <= 3 and not args.no_brute:
        rb = measure(kmb, kmlib, torch, w, dev, stream, kmb.KM_MODE_BRUTE, 1, 1, args.variant, instrument=True)
        brute = {"ms_per_iter": rb["ms_per_iter"], "distances_per_s": n * k / (rb["ms_per_iter"] * 1e-3),
                 "roofline": kernel_roofline(w, rb, 1, nsm, hbm), "identical_sse": rb["sse"] == r["sse"]}

    cpu = None
    if not args.no_cpu_baseline and rank == 0:
        cpu = cpu_baseline(w, args.cpu_seconds)

    st = r["stats"]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": K, "warmup": W,
        "ms_per_step": r["ms_per_step"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": ("tf32x3 tensor scores / f64 certify / int64 sums" if d > 3 else
                  "f32 scan / f64 certify / int64 sums"), "data": "synthetic",
        "config": {"workload": w.name, "desc": w.desc, "n": n, "d": d, "k": k, "iterations_per_step": T,
                   "mode": args.mode, "path": "tiles" if st["tiles"] else "brute",
                   "step": f"one km_run_ctx call = the config's full run: {T} Lloyd iterations (tol=-1), "
                           "index build, final SSE and labels in input order included",
                   "l2": "no flush: per-iteration working set points+labels = %d MB > 126 MB L2" %
                         ((n * d * 4 + n * 4) >> 20),
                   "assign_variant": args.variant if args.variant is not None else "default"},
        "ms_per_iter": r["ms_per_iter"],
        "ms_per_step_median": r["ms_per_step_median"], "ms_per_step_min": r["ms_per_step_min"],
        "ms_per_iter_median": r["ms_per_step_median"] / T,
        "distances_per_s": value,
        "roofline_fraction_step_vs_bruteforce_fp32": (3.0 * d * n * k / (r["ms_per_iter"] * 1e-3) / 1e12) /
                                                     _peak_fp32(nsm),
        "fp32_peaks": {"nominal_tflops_at_max_clock": _peak_fp32(nsm),
                       "at_measured_clock_tflops": _peak_fp32(nsm, clocks["sm_mhz"]) if clocks.get("sm_mhz") else None,
                       "measured_ffma_probe_tflops": measured_fp32_peak(),
                       "note": "SM count x 128 lanes x 2 FLOP x clock; probe = tools/fp32_probe.cu on this pool "
                               "(profiles/r01/fp32_probe.jsonl)"},
        "roofline": roof,
        "breakdown": breakdown,
        "work": {"pairs_evaluated_per_iter": st["pairs"] / T, "bruteforce_pairs_per_iter": n * k,
                 "points_scanned_per_iter": st["points_scanned"] / T, "batch_tiles_per_iter": st["batch_tiles"] / T,
                 "listed_tiles_per_iter": st["tile_visits"] / T, "eq5_tiles_per_iter": st["eq5_tiles"] / T,
                 "eq4_tiles_per_iter": st["eq4_tiles"] / T, "changed_t": r["changed_t"]},
        "brute_force": brute,
        "hd_decisions": hd_stats,
        "gpu_launches": r["launches"],
        "e2e": {"value": e2e_val, "unit": UNIT, "ms_per_step": re["ms_per_step"],
                "h2d_bytes_per_step": n * d * 4 + k * d * 4, "d2h_bytes_per_step": n * 4 + k * d * 4 + 8 + 8,
                "note": "km_run_ctx with pinned host buffers: points/C0 H2D, labels/centroids/SSE D2H every step"},
        "clocks": clocks,
        "cpu_baseline": cpu,
        "sse": r["sse"],
    }
    print(json.dumps(line), flush=True)
    return 0


def run_native_dp(args, world, rank, local):
    import torch
    from paper_2412_02244_b200 import dp
    dev = torch.device("cuda", local)
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    hbm = peaks().get("hbm_gbs", 6650.0)
    extras = {"sampler": ClockSampler,
              "roofline": lambda w, r, K: kernel_roofline(w, r, K, nsm, hbm)}
    return dp.bench_dp(args, world, rank, local, synth, METRIC, UNIT, extras)


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_native(args)


if __name__ == "__main__":
    sys.exit(main())
