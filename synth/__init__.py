"""synth -- seeded synthetic spatial-vector workloads (inputs only, no k-means arithmetic).

Shared by tests/, bench.py and smoke(): this module is the ONLY code both the
oracle side and the CUDA side see, and it holds none of the method's arithmetic
(no distances, no argmin, no means) -- it only draws points and initial centroids.

The paper's datasets (PAPER.md Table `tab:datasets`: T-drive, Porto,
Argo-AVL 2-D geo-locations; Argo-PC, 3D-RD, Shapenet 3-D point clouds) are not
available; these generators stand in for them with the shapes, sizes and
structure BASELINE.json's ``configs`` name (recipe: DESIGN.md "Inputs",
SURVEY.md section 8(d)).

Common rules: ``numpy.random.default_rng(seed)`` (PCG64); draws in float64, then
``astype(float32)`` (round to nearest); points shuffled with ``rng.permutation``;
initial centroids C0 = P[rng.choice(n, k, replace=False)] drawn afterwards from
the same stream (config 1: first k points, no shuffle).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Workload:
    name: str
    points: np.ndarray     # float32 [n][d], C-contiguous
    init: np.ndarray       # float32 [k][d]
    iters: int
    desc: str

    @property
    def n(self):
        return self.points.shape[0]

    @property
    def d(self):
        return self.points.shape[1]

    @property
    def k(self):
        return self.init.shape[0]


def _finish(rng, P64, k, shuffle=True):
    P = np.ascontiguousarray(P64.astype(np.float32))
    if shuffle:
        P = np.ascontiguousarray(P[rng.permutation(P.shape[0])])
    idx = rng.choice(P.shape[0], k, replace=False)
    return P, np.ascontiguousarray(P[idx])


def uniform_unit(n=10_000, d=2, k=10, seed=0):
    """Config 1: uniform in [0,1)^d sampled directly in float32; C0 = first k points."""
    rng = np.random.default_rng(seed)
    P = np.ascontiguousarray(rng.random((n, d), dtype=np.float32))
    return P, np.ascontiguousarray(P[:k].copy())


def geo_gaussians(n=1_000_000, k=100, n_comp=50, seed=0, shuffle=True):
    """Config 2: 2-D lon/lat mixture of isotropic Gaussians (equal counts).

    means ~ U([-180,180) x [-90,90)), sigma ~ U[0.1, 2); no clipping."""
    rng = np.random.default_rng(seed)
    mu = np.stack([rng.uniform(-180, 180, n_comp), rng.uniform(-90, 90, n_comp)], axis=1)
    sig = rng.uniform(0.1, 2.0, n_comp)
    parts = []
    for c, cnt in enumerate(np.diff(np.linspace(0, n, n_comp + 1).round().astype(np.int64))):
        parts.append(mu[c] + sig[c] * rng.standard_normal((cnt, 2)))
    return _finish(rng, np.concatenate(parts), k, shuffle)


def _plane(rng, cnt):
    centre = rng.uniform(-28, 28, 3)
    nrm = rng.standard_normal(3)
    nrm /= np.linalg.norm(nrm)
    a = rng.standard_normal(3)
    u = a - (a @ nrm) * nrm
    u /= np.linalg.norm(u)
    v = np.cross(nrm, u)
    Lu, Lv = rng.uniform(5, 30, 2)
    s = rng.uniform(-Lu / 2, Lu / 2, cnt)
    t = rng.uniform(-Lv / 2, Lv / 2, cnt)
    return centre + s[:, None] * u + t[:, None] * v


def _sphere(rng, cnt):
    centre = rng.uniform(-45, 45, 3)
    r = rng.uniform(0.5, 5.0)
    g = rng.standard_normal((cnt, 3))
    g /= np.linalg.norm(g, axis=1, keepdims=True)
    return centre + r * g


def point_cloud(n=1_000_000, k=1000, n_planes=20, n_spheres=10, seed=0, shuffle=True):
    """Configs 3/4: 3-D points on random planes and spheres in [-50,50]^3 + N(0, 0.02^2) noise.

    n is split with array_split over the surfaces, planes first."""
    rng = np.random.default_rng(seed)
    counts = [len(a) for a in np.array_split(np.arange(n), n_planes + n_spheres)]
    parts = []
    for s, cnt in enumerate(counts):
        parts.append(_plane(rng, cnt) if s < n_planes else _sphere(rng, cnt))
    P = np.concatenate(parts)
    P += rng.normal(0.0, 0.02, P.shape)
    return _finish(rng, P, k, shuffle)


def big_mixture(n=100_000_000, k=10_000, n_comp=500, bg_frac=0.1, seed=0, shuffle=True):
    """Config 5: 2-D mixture of Gaussians (sigma ~ U[0.28, 5.6)) + uniform background in [0,1000)^2."""
    rng = np.random.default_rng(seed)
    n_bg = int(round(n * bg_frac))
    n_g = n - n_bg
    mu = rng.uniform(0, 1000, (n_comp, 2))
    sig = rng.uniform(0.28, 5.6, n_comp)
    out = np.empty((n, 2), np.float32)
    cuts = np.linspace(0, n_g, n_comp + 1).round().astype(np.int64)
    for c in range(n_comp):
        a, b = cuts[c], cuts[c + 1]
        out[a:b] = (mu[c] + sig[c] * rng.standard_normal((b - a, 2))).astype(np.float32)
    out[n_g:] = rng.uniform(0, 1000, (n_bg, 2)).astype(np.float32)
    if shuffle:
        out = out[rng.permutation(n)]
    out = np.ascontiguousarray(out)
    idx = rng.choice(n, k, replace=False)
    return out, np.ascontiguousarray(out[idx])


# BASELINE.json "configs", in order.  scale < 1 shrinks n (and k proportionally
# only if keep_k is False) for oracle-sized samples of the same distribution.
CONFIGS = {
    1: dict(desc="n=1e4 d=2 k=10 uniform [0,1)^2, C0 = first k, 10 iters", iters=10),
    2: dict(desc="n=1e6 d=2 k=100 mixture of 50 Gaussians (lon/lat), 20 iters", iters=20),
    3: dict(desc="n=1e6 d=3 k=1000 20 planes + 10 spheres, 20 iters", iters=20),
    4: dict(desc="n=1e7 d=3 k=1000 133 planes + 67 spheres (headline), 20 iters", iters=20),
    5: dict(desc="n=1e8 d=2 k=1e4 500 Gaussians + 10% uniform in [0,1000)^2, 10 iters", iters=10),
    # NEXT-4: the paper's high-dimensional check (Table tab:high_dimension)
    6: dict(desc="n=5e5 d=128 k=1000 embedded trajectories (Apoll-TD stand-in), 20 iters", iters=20),
    7: dict(desc="n=5e5 d=256 k=1000 embedded trajectories (Argo-ETD stand-in), 20 iters", iters=20),
}


def embedded_trajectories(n=500_000, d=128, k=1000, n_routes=200, seed=0, shuffle=True):
    """NEXT-4 stand-in for Apoll-TD (d=128) / Argo-ETD (d=256), "trajectory data embedded
    into fixed-length vectors" (Table tab:datasets): a trajectory is d/2 planar
    positions (x_0, y_0, ..., x_{d/2-1}, y_{d/2-1}) flattened.  n_routes smooth routes (start
    U[-50,50)^2, heading U[0,2pi), speed U[0.5,2), turn rate N(0, 0.05^2) per step); each
    trajectory follows a random route with an offset N(0, 2^2) per axis, a speed factor
    U[0.8,1.25) and per-position noise N(0, 0.3^2).  Equal-probability routes; not centred."""
    rng = np.random.default_rng(seed)
    T = d // 2
    start = rng.uniform(-50, 50, (n_routes, 2))
    head = rng.uniform(0, 2 * np.pi, n_routes)
    speed = rng.uniform(0.5, 2.0, n_routes)
    turn = rng.normal(0, 0.05, (n_routes, T))
    ang = head[:, None] + np.cumsum(turn, axis=1)
    route = rng.integers(0, n_routes, n)
    P64 = np.empty((n, T, 2))
    step = np.stack([np.cos(ang), np.sin(ang)], -1) * speed[:, None, None]      # [R][T][2]
    prog = np.arange(T, dtype=np.float64)
    for r0 in range(0, n, 65536):   # chunked: bounded temporaries
        r = route[r0:r0 + 65536]
        m = len(r)
        f = rng.uniform(0.8, 1.25, m)
        off = rng.normal(0, 2.0, (m, 1, 2))
        # position t = start + f * sum_{u < t} step_u
        cs = np.cumsum(step[r], axis=1) - step[r]
        P64[r0:r0 + m] = start[r][:, None, :] + f[:, None, None] * cs + off + rng.normal(0, 0.3, (m, T, 2))
    del prog
    return _finish(rng, P64.reshape(n, d), k, shuffle)


def config(i: int, n: int | None = None, k: int | None = None, seed: int = 0) -> Workload:
    """Workload for BASELINE.json config i (1-based); n/k override the size only."""
    c = CONFIGS[i]
    if i == 1:
        P, C0 = uniform_unit(n or 10_000, 2, k or 10, seed)
    elif i == 2:
        P, C0 = geo_gaussians(n or 1_000_000, k or 100, 50, seed)
    elif i == 3:
        P, C0 = point_cloud(n or 1_000_000, k or 1000, 20, 10, seed)
    elif i == 4:
        P, C0 = point_cloud(n or 10_000_000, k or 1000, 133, 67, seed)
    elif i == 5:
        P, C0 = big_mixture(n or 100_000_000, k or 10_000, 500, 0.1, seed)
    elif i == 6:
        P, C0 = embedded_trajectories(n or 500_000, 128, k or 1000, seed=seed)
    elif i == 7:
        P, C0 = embedded_trajectories(n or 500_000, 256, k or 1000, seed=seed)
    else:
        raise KeyError(i)
    return Workload(f"config{i}", P, C0, c["iters"], c["desc"])


def random_instance(seed: int, n: int, d: int, k: int, kind: str = "blobs"):
    """Small seeded parity instance: points + k distinct-index initial centroids."""
    rng = np.random.default_rng(seed)
    if kind == "uniform":
        P = rng.uniform(-10, 10, (n, d))
    elif kind == "grid":          # integer lattice: many exact distance ties
        P = rng.integers(-4, 5, (n, d)).astype(np.float64)
    elif kind == "offset":        # far from the origin: punishes expanded-form shortcuts
        P = 1.0e4 + rng.normal(0, 1.0, (n, d))
    else:
        nb = max(1, k // 2)
        mu = rng.uniform(-20, 20, (nb, d))
        P = mu[rng.integers(0, nb, n)] + rng.normal(0, 1.5, (n, d))
    P = np.ascontiguousarray(P.astype(np.float32))
    idx = rng.choice(n, k, replace=False)
    return P, np.ascontiguousarray(P[idx])
