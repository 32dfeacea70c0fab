"""Thin ctypes binding of libkm (include/km.h): argument marshalling only.

Every step of the Lloyd path runs in libkm's sm_100a kernels; this module only
turns torch tensors / numpy arrays into pointers, passes the current torch CUDA
stream, and maps status codes to exceptions.  There is no CPU fallback: if
libkm.so is missing the import fails loudly.

Names follow km.h: km_create, km_destroy, km_assign, km_update, km_run,
km_run_ctx, km_read_traces, km_timing_*, km_launch_count.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KM_LIB_PATH") or os.path.join(_HERE, "libkm.so")   # override: tuning builds

KM_OK, KM_E_INVALID, KM_E_UNSUPPORTED, KM_E_NOMEM, KM_E_CUDA, KM_E_STATE = 0, -1, -2, -3, -4, -5


class KmError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        msg = _lib.km_strerror(code).decode() if _lib is not None else str(code)
        if code == KM_E_CUDA:
            msg += f" (cudaError {_lib.km_last_cuda_error()})"
        super().__init__(f"{where}: {msg} [{code}]")


class _Timing(ctypes.Structure):
    _fields_ = [("assign_ms", ctypes.c_double), ("update_ms", ctypes.c_double), ("other_ms", ctypes.c_double),
                ("assign_launches", ctypes.c_int64), ("update_launches", ctypes.c_int64),
                ("other_launches", ctypes.c_int64)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libkm.so not built at {LIB_PATH}: run `make` (or __graft_entry__.build()); "
                          "there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    V, I64, I32, F, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_float, ctypes.c_double
    sig = {
        "km_create": ([ctypes.POINTER(V), I64, I32, I32, V], ctypes.c_int),
        "km_destroy": ([V], ctypes.c_int),
        "km_set_stream": ([V, V], ctypes.c_int),
        "km_max_k": ([I32], I32),
        "km_assign": ([V, V, V, V, V], ctypes.c_int),
        "km_update": ([V, V, V, V, V, V, V], ctypes.c_int),
        "km_run_ctx": ([V, V, V, I32, F, V, V, ctypes.POINTER(D), V, V], ctypes.c_int),
        "km_run": ([V, I64, I32, I32, V, I32, F, V, V, ctypes.POINTER(D)], ctypes.c_int),
        "km_read_traces": ([V, V, V, V, I32], ctypes.c_int),
        "km_timing_enable": ([V, ctypes.c_int], ctypes.c_int),
        "km_timing_read": ([V, ctypes.POINTER(_Timing), ctypes.c_int], ctypes.c_int),
        "km_launch_count": ([V, ctypes.c_int], I64),
        "km_strerror": ([ctypes.c_int], ctypes.c_char_p),
        "km_last_cuda_error": ([], ctypes.c_int),
        "km_set_mode": ([V, ctypes.c_int], ctypes.c_int),
        "km_dp_bbox": ([V, V, V], ctypes.c_int),
        "km_dp_begin": ([V, V, V, V, I64, I32], ctypes.c_int),
        "km_dp_partial_len": ([V], I64),
        "km_dp_step": ([V, V], ctypes.c_int),
        "km_dp_apply": ([V, V, F, ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
        "km_dp_end": ([V, V, V, ctypes.POINTER(D), V], ctypes.c_int),
        "km_dp_sse": ([V, V], D),
        "km_debug_stats": ([V, V], ctypes.c_int),
        "km_read_stats": ([V, V], ctypes.c_int),
        "km_debug_set_variant": ([V, ctypes.c_int], ctypes.c_int),
        "km_debug_assign_grid": ([V], ctypes.c_int),
        "km_debug_set": ([V, ctypes.c_int, ctypes.c_int], ctypes.c_int),
        "km_hd_stats": ([V, V], ctypes.c_int),
        "km_debug_bounds": ([V, V], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    return lib


_lib = _load()

EXPORTED = ["km_create", "km_destroy", "km_set_stream", "km_max_k", "km_assign", "km_update", "km_run_ctx",
            "km_run", "km_read_traces", "km_timing_enable", "km_timing_read", "km_launch_count", "km_strerror",
            "km_last_cuda_error", "km_set_mode", "km_read_stats", "km_dp_bbox", "km_dp_begin", "km_dp_partial_len", "km_dp_step",
            "km_dp_apply", "km_dp_end", "km_dp_sse", "km_debug_stats", "km_debug_set_variant", "km_debug_assign_grid", "km_debug_set",
            "km_hd_stats", "km_debug_bounds"]

KM_MODE_AUTO, KM_MODE_BRUTE, KM_MODE_TILES, KM_MODE_BOUNDS = 0, 1, 2, 3


def _check(rc: int, where: str) -> int:
    if rc < 0:
        raise KmError(rc, where)
    return rc


def _ptr(x, dtype=None):
    """Pointer of a torch tensor (CPU or CUDA) or numpy array; None -> NULL."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        if dtype is not None and x.dtype != np.dtype(dtype):
            raise TypeError(f"expected {dtype}, got {x.dtype}")
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return ctypes.c_void_p(x.ctypes.data)
    import torch
    if isinstance(x, torch.Tensor):
        tmap = {np.float32: torch.float32, np.int32: torch.int32, np.float64: torch.float64, np.int64: torch.int64}
        if dtype is not None and x.dtype != tmap[np.dtype(dtype).type]:
            raise TypeError(f"expected {dtype}, got {x.dtype}")
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return ctypes.c_void_p(x.data_ptr())
    if isinstance(x, int):
        return ctypes.c_void_p(x)
    raise TypeError(f"unsupported argument type {type(x)}")


def _current_stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def km_max_k(d: int) -> int:
    return int(_lib.km_max_k(d))


def km_create(n: int, d: int, k: int, stream=None):
    h = ctypes.c_void_p()
    s = _current_stream() if stream is None else ctypes.c_void_p(stream)
    _check(_lib.km_create(ctypes.byref(h), n, d, k, s), "km_create")
    return h


def km_destroy(ctx) -> None:
    _check(_lib.km_destroy(ctx), "km_destroy")


def km_set_stream(ctx, stream=None) -> None:
    s = _current_stream() if stream is None else ctypes.c_void_p(stream)
    _check(_lib.km_set_stream(ctx, s), "km_set_stream")


def km_assign(ctx, points, centroids, labels, sse_dev=None) -> None:
    _check(_lib.km_assign(ctx, _ptr(points, np.float32), _ptr(centroids, np.float32), _ptr(labels, np.int32),
                          _ptr(sse_dev, np.float64)), "km_assign")


def km_update(ctx, points, labels, old_centroids, new_centroids, counts=None, max_drift_dev=None) -> None:
    _check(_lib.km_update(ctx, _ptr(points, np.float32), _ptr(labels, np.int32), _ptr(old_centroids, np.float32),
                          _ptr(new_centroids, np.float32), _ptr(counts, np.int32), _ptr(max_drift_dev, np.float64)),
           "km_update")


def km_run_ctx(ctx, points, init_centroids, max_iter: int, tol: float, out_centroids, out_labels,
               sse_trace_dev=None, changed_trace_dev=None):
    """Returns (iterations, out_sse)."""
    sse = ctypes.c_double(0.0)
    it = _check(_lib.km_run_ctx(ctx, _ptr(points, np.float32), _ptr(init_centroids, np.float32), int(max_iter),
                                float(tol), _ptr(out_centroids, np.float32), _ptr(out_labels, np.int32),
                                ctypes.byref(sse), _ptr(sse_trace_dev, np.float64),
                                _ptr(changed_trace_dev, np.int64)), "km_run_ctx")
    return it, sse.value


def km_run(points, n: int, d: int, k: int, init_centroids, max_iter: int, tol: float, out_centroids, out_labels):
    """The north-star signature; returns (iterations, out_sse)."""
    sse = ctypes.c_double(0.0)
    it = _check(_lib.km_run(_ptr(points, np.float32), int(n), int(d), int(k), _ptr(init_centroids, np.float32),
                            int(max_iter), float(tol), _ptr(out_centroids, np.float32), _ptr(out_labels, np.int32),
                            ctypes.byref(sse)), "km_run")
    return it, sse.value


@dataclass
class Traces:
    sse: np.ndarray
    changed: np.ndarray
    max_drift: np.ndarray


def km_read_traces(ctx, count: int) -> Traces:
    s = np.zeros(count, np.float64)
    c = np.zeros(count, np.int64)
    m = np.zeros(count, np.float64)
    it = _check(_lib.km_read_traces(ctx, _ptr(s), _ptr(c), _ptr(m), count), "km_read_traces")
    it = min(it, count)
    return Traces(s[:it], c[:it], m[:it])


def km_timing_enable(ctx, on: bool = True) -> None:
    _check(_lib.km_timing_enable(ctx, int(bool(on))), "km_timing_enable")


def km_timing_read(ctx, reset: bool = False) -> dict:
    t = _Timing()
    _check(_lib.km_timing_read(ctx, ctypes.byref(t), int(bool(reset))), "km_timing_read")
    return {f: getattr(t, f) for f, _ in _Timing._fields_}


def km_launch_count(ctx, reset: bool = False) -> int:
    return int(_lib.km_launch_count(ctx, int(bool(reset))))


def km_set_mode(ctx, mode: int) -> None:
    """KM_MODE_AUTO / KM_MODE_BRUTE / KM_MODE_TILES / KM_MODE_BOUNDS (identical results; see km.h)."""
    _check(_lib.km_set_mode(ctx, int(mode)), "km_set_mode")


def km_read_stats(ctx) -> dict:
    out = np.zeros(4, np.int64)
    tiles = _check(_lib.km_read_stats(ctx, _ptr(out)), "km_read_stats")
    r = {"tiles": bool(tiles), "pairs": int(out[0]), "points_scanned": int(out[1]), "batch_tiles": int(out[2]),
         "tile_visits": int(out[3]), "eq5_tiles": 0, "eq4_tiles": 0, "split_tiles": 0,
         "l1_list_len": 0, "l1_nodes": 0, "tile_cands": 0, "ovf_tiles": 0, "l1_long_nodes": 0}
    if tiles:
        s32 = km_debug_stats(ctx)
        r["eq5_tiles"] = int(s32[12])    # tiles settled by the node inter bound (Eq. 5) in tile_filter_kernel
        r["eq4_tiles"] = int(s32[13])    # K1t: listed tiles whose every point passed Eq. 4
        r["split_tiles"] = int(s32[29])  # K1t: listed tiles pruned with their two sub-balls (split at a Morton jump)
        r["l1_list_len"] = int(s32[10])  # level-1 prune: summed node-list lengths the tile candidates came from
        r["l1_nodes"] = int(s32[11])     # level-1 prune: nodes
        r["tile_cands"] = int(s32[15])   # level-1 prune: summed per-tile candidate counts
        r["ovf_tiles"] = int(s32[14])    # K1t: listed tiles with more than kTC candidates (overflow pool)
        r["l1_long_nodes"] = int(s32[16])  # level-1 nodes whose tiles went to tile_cands_kernel (long lists)
    return r


def km_dp_bbox(ctx, points) -> np.ndarray:
    """Local bounding box of the shard: float32 [2d] (mins, then maxes)."""
    d = points.shape[1]
    out = np.zeros(2 * d, np.float32)
    _check(_lib.km_dp_bbox(ctx, _ptr(points, np.float32), _ptr(out)), "km_dp_bbox")
    return out


def km_dp_begin(ctx, points, init_centroids, lo_hi, n_global: int, max_iter: int) -> None:
    lo_hi = np.ascontiguousarray(lo_hi, np.float32)
    _check(_lib.km_dp_begin(ctx, _ptr(points, np.float32), _ptr(init_centroids, np.float32), _ptr(lo_hi),
                            int(n_global), int(max_iter)), "km_dp_begin")


def km_dp_partial_len(ctx) -> int:
    """Length of the context's partial (k*d + k + 1; k*d' + 2k + 1 for the high-d variant)."""
    return _check(_lib.km_dp_partial_len(ctx), "km_dp_partial_len")


def km_dp_step(ctx, partial_dev) -> None:
    """partial_dev: int64 CUDA tensor [km_dp_partial_len] (uint64 bit patterns)."""
    _check(_lib.km_dp_step(ctx, _ptr(partial_dev, np.int64)), "km_dp_step")


def km_dp_apply(ctx, partial_dev, tol: float, want_done: bool = False):
    """Returns (iterations applied, done flag or None)."""
    done = ctypes.c_int(0)
    it = _check(_lib.km_dp_apply(ctx, _ptr(partial_dev, np.int64), float(tol),
                                 ctypes.byref(done) if want_done else None), "km_dp_apply")
    return it, (bool(done.value) if want_done else None)


def km_dp_end(ctx, out_centroids, out_labels):
    """Returns (iterations, local Eq. 1 SSE of the shard, its 3 fixed-point limbs as int64 [3])."""
    sse = ctypes.c_double(0.0)
    limbs = np.zeros(3, np.uint64)
    it = _check(_lib.km_dp_end(ctx, _ptr(out_centroids, np.float32), _ptr(out_labels, np.int32), ctypes.byref(sse),
                               _ptr(limbs)), "km_dp_end")
    return it, sse.value, limbs.astype(np.int64)


def km_dp_sse(ctx, limbs_sum) -> float:
    """Eq. 1 over all ranks from the limb-wise sum of every rank's km_dp_end limbs."""
    a = np.ascontiguousarray(np.asarray(limbs_sum).astype(np.int64)).view(np.uint64)
    return float(_lib.km_dp_sse(ctx, _ptr(a)))


def km_debug_stats(ctx) -> np.ndarray:
    out = np.zeros(32, np.int64)
    _check(_lib.km_debug_stats(ctx, _ptr(out)), "km_debug_stats")
    return out


def km_hd_stats(ctx) -> dict:
    """High-dimensional variant: how the assignments of the last run were decided (cumulative
    over its iterations): certified from the tensor-core top 2, FP64 among the top-4 band,
    FP64 over all k."""
    out = np.zeros(3, np.int64)
    _check(_lib.km_hd_stats(ctx, _ptr(out)), "km_hd_stats")
    return {"certified": int(out[0]), "band": int(out[1]), "full_scan": int(out[2])}


def km_debug_set_variant(ctx, variant: int) -> None:
    """0 = simple per-pair top-2 scan, 1 = packed FP32x2 scan (default)."""
    _check(_lib.km_debug_set_variant(ctx, int(variant)), "km_debug_set_variant")


def km_debug_assign_grid(ctx) -> int:
    return int(_lib.km_debug_assign_grid(ctx))


KM_DBG_ST_SHIFT, KM_DBG_K1T_MINB, KM_DBG_HD, KM_DBG_GRAPH, KM_DBG_SMALL, KM_DBG_PDL, KM_DBG_SHORT_LIST = 1, 2, 3, 4, 5, 6, 7


def km_debug_bounds(ctx) -> np.ndarray:
    """KM_MODE_BOUNDS counters of the last run (km.h km_debug_bounds): int64 [8]."""
    out = np.zeros(8, np.int64)
    _check(_lib.km_debug_bounds(ctx, _ptr(out)), "km_debug_bounds")
    return out


def km_debug_set(ctx, what: int, value: int) -> None:
    """Per-context test/tuning override (km.h km_debug_set)."""
    _check(_lib.km_debug_set(ctx, int(what), int(value)), "km_debug_set")


class Context:
    """RAII holder of a km_ctx (create on construction, destroy on close/GC)."""

    def __init__(self, n: int, d: int, k: int, stream=None):
        self.n, self.d, self.k = n, d, k
        self.handle = km_create(n, d, k, stream)

    def close(self):
        if self.handle is not None:
            km_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
