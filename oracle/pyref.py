"""oracle.pyref -- Lloyd's algorithm in exact rational arithmetic, pure Python.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  For tiny inputs; it pins the
C oracle.  Every value is a ``fractions.Fraction``, so there is no rounding at
all: distances, ties, means and SSE are the mathematical values.

Follows PAPER.md: Eq. 1 objective, assignment to the nearest centroid
(P:L99), refine c_j <- sv(j)/|S_j| (Alg. 1 line 12), loop until no centroid
moves.  Ties -> lowest index; empty cluster keeps its centroid
(readings R2, R5).
"""
from __future__ import annotations

from fractions import Fraction


def _F(x):
    return x if isinstance(x, Fraction) else Fraction(x)


def sqdist(p, c):
    return sum((_F(a) - _F(b)) ** 2 for a, b in zip(p, c))


def assign(points, centroids):
    labels = []
    best = []
    for p in points:
        b, a = None, None
        for j, c in enumerate(centroids):
            D = sqdist(p, c)
            if b is None or D < b:
                b, a = D, j
        labels.append(a)
        best.append(b)
    return labels, best


def update(points, labels, centroids):
    k, d = len(centroids), len(centroids[0])
    sums = [[Fraction(0)] * d for _ in range(k)]
    cnt = [0] * k
    for p, j in zip(points, labels):
        cnt[j] += 1
        for m in range(d):
            sums[j][m] += _F(p[m])
    new = []
    for j in range(k):
        if cnt[j]:
            new.append([s / cnt[j] for s in sums[j]])
        else:
            new.append([_F(v) for v in centroids[j]])
    return new, cnt


def sse(points, labels, centroids):
    return sum(sqdist(p, centroids[j]) for p, j in zip(points, labels))


def lloyd(points, c0, max_iter, stop_at_fixpoint=True):
    """Returns (centroids, labels, out_sse, iterations, sse_trace)."""
    C = [[_F(v) for v in c] for c in c0]
    labels, prev, trace = None, None, []
    it = 0
    for t in range(max_iter):
        labels, best = assign(points, C)
        trace.append(sum(best))
        Cn, _ = update(points, labels, C)
        moved = any(a != b for ca, cb in zip(C, Cn) for a, b in zip(ca, cb))
        changed = prev is None or labels != prev
        C, prev, it = Cn, labels, t + 1
        if stop_at_fixpoint and (not moved or (t >= 1 and not changed)):
            break
    return C, labels, sse(points, labels, C), it, trace
