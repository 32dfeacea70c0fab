#!/usr/bin/env python3
"""bench.py -- exact Lloyd step on one B200 (BASELINE.json headline: config 4,
n=1e7 d=3 k=1000), printed as ONE JSON line.

A "step" is one Lloyd iteration (assign + update + convergence bookkeeping) over
the whole synthetic workload.  `--steps K` timed iterations run as one km_run_ctx
call with max_iter = K, tol = -1 (fixed count); `--warmup W` iterations run first.

value  = point-centroid distances/s = n*k*K / device time (CUDA events on the
         library's stream), inputs already resident in HBM.
e2e    = same metric through km_run_ctx with PINNED HOST buffers (H2D of points
         and C0, D2H of labels, centroids and SSE inside the timed region).
roofline: the assignment kernel (dominant), FP32 CUDA-core bound ("alu"):
         achieved = 3*d*n*k FLOP per launch / mean launch time (events around
         every launch inside libkm), peak = 148 SM x 128 lanes x 2 x 1.965 GHz.
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
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--variant", type=int, default=None, help="assign kernel variant (debug)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="oracle sample budget")
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


def run_native(args):
    import torch
    import paper_2412_02244_b200 as kmb
    from paper_2412_02244_b200 import km as kmlib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        return run_native_dp(args, world, rank, local)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    w = synth.config(args.config)
    n, d, k = w.n, w.d, w.k
    K, W = args.steps, max(args.warmup, 3)
    stream = torch.cuda.current_stream(dev)

    Pd = torch.from_numpy(w.points).to(dev)
    C0d = torch.from_numpy(w.init).to(dev)
    Cout = torch.empty((k, d), dtype=torch.float32, device=dev)
    lab = torch.empty(n, dtype=torch.int32, device=dev)
    ctx = kmb.Context(n, d, k, stream.cuda_stream)
    if args.variant is not None:
        kmlib.km_debug_set_variant(ctx.handle, args.variant)

    # warm-up (untimed)
    kmb.km_run_ctx(ctx.handle, Pd, C0d, W, -1.0, Cout, lab)
    torch.cuda.synchronize()

    # timed: exactly K iterations, device-resident inputs
    kmb.km_timing_enable(ctx.handle, True)
    kmb.km_timing_read(ctx.handle, reset=True)
    kmb.km_launch_count(ctx.handle, reset=True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    torch.cuda.synchronize()
    with sampler:
        ev0.record(stream)
        it, sse = kmb.km_run_ctx(ctx.handle, Pd, C0d, K, -1.0, Cout, lab)
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = kmb.km_launch_count(ctx.handle)
    tm = kmb.km_timing_read(ctx.handle, reset=True)
    kmb.km_timing_enable(ctx.handle, False)
    total_ms = ev0.elapsed_time(ev1)
    assert it == K
    ms_iter = total_ms / K
    value = n * k / (ms_iter * 1e-3)

    # roofline of the dominant kernel (assignment): 3*d FLOP per point-centroid pair
    a_ms = tm["assign_ms"] / max(tm["assign_launches"], 1)
    flops = 3.0 * d * n * k
    achieved = flops / (a_ms * 1e-3) / 1e12
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    peak = nsm * FP32_LANES_PER_SM * 2 * SM_MAX_MHZ_NOMINAL * 1e6 / 1e12
    clocks = sampler.summary()
    peak_at_clock = None
    if clocks.get("sm_mhz"):
        peak_at_clock = nsm * FP32_LANES_PER_SM * 2 * clocks["sm_mhz"] * 1e6 / 1e12

    # e2e: pinned host buffers through the same public call
    Ph = torch.from_numpy(w.points).pin_memory()
    C0h = torch.from_numpy(w.init).pin_memory()
    Ch = torch.empty((k, d), dtype=torch.float32).pin_memory()
    lh = torch.empty(n, dtype=torch.int32).pin_memory()
    kmb.km_run_ctx(ctx.handle, Ph, C0h, W, -1.0, Ch, lh)   # allocates the staging buffers once
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    it2, sse2 = kmb.km_run_ctx(ctx.handle, Ph, C0h, K, -1.0, Ch, lh)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    e2e_val = n * k * K / (e2e_ms * 1e-3)
    assert sse2 == sse, (sse2, sse)
    ctx.close()

    cpu = None
    if not args.no_cpu_baseline and rank == 0:
        cpu = cpu_baseline(w, args.cpu_seconds)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": K, "warmup": W,
        "ms_per_step": ms_iter, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 scan / f64 certify+sums", "data": "synthetic",
        "config": {"workload": w.name, "desc": w.desc, "n": n, "d": d, "k": k,
                   "step": "one Lloyd iteration (assign+update+finalize), tol=-1",
                   "l2": "no flush: per-iteration working set points+labels = %d MB > 126 MB L2" %
                         ((n * d * 4 + n * 4) >> 20),
                   "assign_kernel": "fast" if args.variant in (None, 1) else "simple"},
        "ms_per_iter": ms_iter,
        "distances_per_s": value,
        "roofline_fraction_step": (flops / (ms_iter * 1e-3) / 1e12) / peak,
        "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic_from_profiles(w.name),
                     "kernel": "assign_fast_kernel (K1)", "flop_per_pair": 3 * d,
                     "peak_note": f"{nsm} SM x 128 FP32 lanes x 2 FLOP x 1965 MHz (nominal max clock); "
                                  "FP32 CUDA-core work, not a tensor-core contraction",
                     "peak_at_measured_clock": peak_at_clock,
                     "frac_at_measured_clock": achieved / peak_at_clock if peak_at_clock else None,
                     "assign_ms_per_launch": a_ms,
                     "update_ms_per_launch": tm["update_ms"] / max(tm["update_launches"], 1),
                     "assign_share_of_step": tm["assign_ms"] / total_ms},
        "gpu_launches": launches,
        "e2e": {"value": e2e_val, "unit": UNIT, "ms_total": e2e_ms, "iterations": K,
                "h2d_bytes_per_step": (n * d * 4 + k * d * 4) / K,
                "d2h_bytes_per_step": (n * 4 + k * d * 4 + 8 + 8) / K,
                "note": "one km_run_ctx call of K iterations with pinned host buffers; bytes amortised per step"},
        "clocks": clocks,
        "cpu_baseline": cpu,
        "sse": sse,
    }
    print(json.dumps(line), flush=True)
    return 0


def run_native_dp(args, world, rank, local):
    from paper_2412_02244_b200 import dp
    return dp.bench_dp(args, world, rank, local, synth, METRIC, UNIT)


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_native(args)


if __name__ == "__main__":
    sys.exit(main())
