"""oracle -- plain, slow, obviously-correct CPU Lloyd (k-means) for parity checks.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2412_02244_b200``) never imports it and
shares no code with it ("Oracle").

Two implementations, both following PAPER.md (P:Lnn = /root/reference/PAPER.md
line nn):

* ``liboracle.so`` (``lloyd_oracle.c``): FP64 plain Lloyd -- Eq. 1,
  nearest-centroid assignment, refine c_j <- sv(j)/|S_j| (Alg. 1 line 12,
  P:L296-299), drift, "until no centroid moves".
* ``pyref`` (pure Python, exact rationals) for tiny inputs; it pins the C code.

Mode A (``round_f32=True``, the parity gate) rounds centroids to float32 between
iterations (reading R8); mode B keeps FP64 (equals scipy's kmeans2).

Every function here is pinned by ``tests/test_oracle_pins.py`` against hand-worked
examples (``tests/golden/``), exact rational arithmetic, scipy/sklearn special
cases and invariants.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lloyd_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

# The oracle's own build line: no -ffast-math, no FMA contraction (the order of
# operations written in lloyd_oracle.c is the definition).
CFLAGS = ["-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (idempotent)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, _SRC, "-o", _LIB + ".tmp", "-lm"])
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        i64, i32, dbl = ctypes.c_int64, ctypes.c_int, ctypes.c_double
        lib.oracle_assign.argtypes = [P, i64, i32, P, i32, P, P, P, i32]
        lib.oracle_assign.restype = None
        lib.oracle_update.argtypes = [P, i64, i32, P, i32, P, P, P, P, i32]
        lib.oracle_update.restype = dbl
        lib.oracle_sse.argtypes = [P, i64, i32, P, P]
        lib.oracle_sse.restype = dbl
        lib.oracle_lloyd.argtypes = [P, i64, i32, i32, P, i32, dbl, i32, P, P, P, P, P, P, i32]
        lib.oracle_lloyd.restype = i32
        lib.oracle_max_threads.argtypes = []
        lib.oracle_max_threads.restype = i32
        _lib = lib
    return _lib


def _ptr(a: np.ndarray) -> ctypes.c_void_p:
    return ctypes.c_void_p(a.ctypes.data)


def _points(P) -> np.ndarray:
    P = np.ascontiguousarray(P, dtype=np.float32)
    if P.ndim != 2:
        raise ValueError("points must be [n][d]")
    return P


def max_threads() -> int:
    return int(_load().oracle_max_threads())


@dataclass
class AssignResult:
    labels: np.ndarray   # int32 [n]
    best: np.ndarray     # float64 [n]  D_{i,a(i)}
    second: np.ndarray   # float64 [n]  min_{j != a(i)} D_ij (inf if k == 1)


def assign(P, C, threads: int = 0) -> AssignResult:
    """Nearest centroid (lowest index on ties) in FP64 direct form."""
    P = _points(P)
    C = np.ascontiguousarray(C, dtype=np.float64)
    n, d = P.shape
    k = C.shape[0]
    lab = np.empty(n, np.int32)
    b1 = np.empty(n, np.float64)
    b2 = np.empty(n, np.float64)
    _load().oracle_assign(_ptr(P), n, d, _ptr(C), k, _ptr(lab), _ptr(b1), _ptr(b2), threads)
    return AssignResult(lab, b1, b2)


@dataclass
class UpdateResult:
    centroids: np.ndarray  # float64 [k][d] (float32-representable in mode A)
    counts: np.ndarray     # int64 [k]
    drift: np.ndarray      # float64 [k]
    max_drift: float


def update(P, labels, C_old, round_f32: bool = True) -> UpdateResult:
    """Refine c_j <- mean of members, empty keeps c_j (Alg. 1 line 12)."""
    P = _points(P)
    lab = np.ascontiguousarray(labels, dtype=np.int32)
    Co = np.ascontiguousarray(C_old, dtype=np.float64)
    n, d = P.shape
    k = Co.shape[0]
    Cn = np.empty_like(Co)
    cnt = np.empty(k, np.int64)
    dr = np.empty(k, np.float64)
    md = _load().oracle_update(_ptr(P), n, d, _ptr(lab), k, _ptr(Co), _ptr(Cn), _ptr(cnt),
                               _ptr(dr), int(bool(round_f32)))
    return UpdateResult(Cn, cnt, dr, float(md))


def sse(P, labels, C) -> float:
    """Eq. 1 of a partition and its centroids, FP64 compensated sum."""
    P = _points(P)
    lab = np.ascontiguousarray(labels, dtype=np.int32)
    C = np.ascontiguousarray(C, dtype=np.float64)
    n, d = P.shape
    return float(_load().oracle_sse(_ptr(P), n, d, _ptr(lab), _ptr(C)))


@dataclass
class LloydResult:
    centroids: np.ndarray      # float64 [k][d]
    labels: np.ndarray         # int32 [n]
    sse: float                 # Eq. 1 of (labels, centroids)
    iterations: int
    sse_trace: np.ndarray      # SSE_t = sum_i min_j D_ij against C_t
    changed_trace: np.ndarray  # changed_t (t = 0 counts n)
    drift_trace: np.ndarray    # max_j Delta_j after iteration t


def lloyd(P, C0, max_iter: int, tol: float = -1.0, round_f32: bool = True,
          threads: int = 0) -> LloydResult:
    """Plain Lloyd from C0 (Alg. 1 skeleton without the index)."""
    P = _points(P)
    C0 = np.ascontiguousarray(C0, dtype=np.float64)
    n, d = P.shape
    k = C0.shape[0]
    if round_f32 and not np.array_equal(C0, C0.astype(np.float32).astype(np.float64)):
        raise ValueError("mode A needs float32-representable initial centroids")
    Cout = np.empty_like(C0)
    lab = np.empty(n, np.int32)
    sse_v = ctypes.c_double(0.0)
    st = np.zeros(max_iter, np.float64)
    ct = np.zeros(max_iter, np.int64)
    dt = np.zeros(max_iter, np.float64)
    it = _load().oracle_lloyd(_ptr(P), n, d, k, _ptr(C0), max_iter, float(tol), int(bool(round_f32)),
                              _ptr(Cout), _ptr(lab), ctypes.byref(sse_v), _ptr(st), _ptr(ct), _ptr(dt),
                              threads)
    return LloydResult(Cout, lab, float(sse_v.value), int(it), st[:it], ct[:it], dt[:it])
