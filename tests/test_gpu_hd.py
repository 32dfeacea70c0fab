"""GPU parity of the high-dimensional variant (d = 32..256): tensor-core
(tcgen05 kind::tf32) scores, exact FP64 certification.

Lockstep: one km_run_ctx iteration from the oracle's float32 centroids C_t; labels must be
IDENTICAL to oracle.assign, the refined centroids within the parity tolerance.  Free runs
against oracle.lloyd (mode A).  The certification paths (top-2 gap, top-4 band in FP64, full
FP64 scan) are all exercised: exact ties (duplicate centroids, lattice data) force the last two.
"""
import numpy as np
import pytest

import oracle
import synth
from helpers import assert_centroids_close, assert_labels_near_tie_only, assert_sse_close

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2412_02244_b200 as kmb  # noqa: E402
from paper_2412_02244_b200 import km as kmlib  # noqa: E402

dev = "cuda"


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def run_ctx(ctx, Pd, C0, iters, tol=-1.0):
    k, d = C0.shape
    Cout = torch.empty((k, d), dtype=torch.float32, device=dev)
    lab = torch.empty(Pd.shape[0], dtype=torch.int32, device=dev)
    it, sse = kmb.km_run_ctx(ctx.handle, Pd, T(np.asarray(C0, np.float32)), iters, tol, Cout, lab)
    tr = kmb.km_read_traces(ctx.handle, iters)
    return it, sse, Cout.cpu().numpy(), lab.cpu().numpy(), tr


def run(P, C0, iters, tol=-1.0):
    n, d = P.shape
    ctx = kmb.Context(n, d, C0.shape[0])
    out = run_ctx(ctx, T(P), C0, iters, tol)
    st = kmlib.km_hd_stats(ctx.handle)
    ctx.close()
    return out + (st,)


def lockstep(P, C0, iters, hd_dbg=0):
    n, d = P.shape
    k = C0.shape[0]
    ctx = kmb.Context(n, d, k)
    if hd_dbg:
        kmlib.km_debug_set(ctx.handle, kmlib.KM_DBG_HD, hd_dbg)
    Pd = T(P)
    C = C0.astype(np.float64)
    for t in range(iters):
        it, sse, Cg, lab_g, tr = run_ctx(ctx, Pd, C, 1)
        assert it == 1
        a = oracle.assign(P, C)
        np.testing.assert_array_equal(lab_g, a.labels, err_msg=f"iteration {t}: labels differ")
        # SSE_t from the exact moment sums: Q - 2 (c - o).S + n ||c - o||^2 per cluster in FP64
        # (quantisation <= 2^-s per coordinate and point, cancellation ~ 2^-52 Q / SSE): 1e-7
        assert_sse_close(tr.sse[0], a.best.sum(), rel=1e-7)
        assert tr.changed[0] == n
        u = oracle.update(P, a.labels, C, round_f32=True)
        assert_centroids_close(Cg, u.centroids, P)
        assert abs(tr.max_drift[0] - u.max_drift) <= 1e-4 * max(u.max_drift, 1e-3 * max(1.0, np.abs(C).max())) + 1e-12
        C = u.centroids
    st = kmlib.km_hd_stats(ctx.handle)
    ctx.close()
    return st


@pytest.mark.parametrize("d", [32, 64, 128, 256])
@pytest.mark.parametrize("n,k", [(1, 1), (130, 7), (3001, 37), (5000, 300)])
def test_hd_lockstep(d, n, k):
    P, C0 = synth.random_instance(7 * n + d + k, n, d, k, "blobs")
    lockstep(P, C0, 3 if n > 1 else 1)


@pytest.mark.parametrize("kind", ["uniform", "offset", "grid"])
def test_hd_lockstep_kinds(kind):
    P, C0 = synth.random_instance(11, 4000, 128, 50, kind)
    lockstep(P, C0, 3)


def test_hd_k_spans_several_centroid_tiles():
    """k = 700: six 128-wide accumulators per point tile, the last one ragged."""
    P, C0 = synth.random_instance(12, 6000, 128, 700, "blobs")
    lockstep(P, C0, 2)


def test_hd_ties_band_and_full_scan():
    """Duplicate centroids tie exactly: 2 copies -> decided in the top-8 band (FP64, lowest j);
    10 copies -> more than 8 in the band -> the FP64 scan over all k.  Labels stay the oracle's."""
    rng = np.random.default_rng(5)
    P = rng.normal(0, 1, (3000, 64)).astype(np.float32)
    base = P[rng.choice(3000, 10, replace=False)]
    C2 = np.concatenate([base, base[:5]])                          # 5 pairs of twins
    C6 = np.concatenate([base[:4]] + [base[4:5]] * 10)             # one centroid 10 times
    for C in (C2, C6):
        ctx = kmb.Context(3000, 64, C.shape[0])
        it, sse, Cg, lab, tr = run_ctx(ctx, T(P), C, 1)
        st = kmlib.km_hd_stats(ctx.handle)
        ctx.close()
        a = oracle.assign(P, C.astype(np.float64))
        np.testing.assert_array_equal(lab, a.labels)
        assert st["band"] + st["full_scan"] > 0
    assert st["full_scan"] > 0


def test_hd_lattice_exact_ties_free_run():
    P, C0 = synth.random_instance(13, 5000, 32, 40, "grid")
    it, sse, C, lab, tr, st = run(P, C0, 6)
    r = oracle.lloyd(P, C0.astype(np.float64), 6, -1.0, True)
    rp = oracle.lloyd(P, C0.astype(np.float64), 5, -1.0, True)
    assert_centroids_close(C, r.centroids, P)
    assert_sse_close(sse, r.sse)
    assert_labels_near_tie_only(P, lab, rp.centroids)
    assert st["band"] + st["full_scan"] > 0


@pytest.mark.parametrize("cfg,n,k,iters", [(6, 20_000, 100, 8), (7, 20_000, 300, 6), (6, 60_000, 1000, 4)])
def test_hd_free_run_configs(cfg, n, k, iters):
    w = synth.config(cfg, n=n, k=k)
    it, sse, C, lab, tr, st = run(w.points, w.init, iters)
    assert it == iters
    r = oracle.lloyd(w.points, w.init.astype(np.float64), iters, -1.0, True)
    rp = oracle.lloyd(w.points, w.init.astype(np.float64), iters - 1, -1.0, True)
    assert_centroids_close(C, r.centroids, w.points)
    assert_sse_close(sse, r.sse)
    assert_labels_near_tie_only(w.points, lab, rp.centroids)
    np.testing.assert_allclose(tr.sse, r.sse_trace, rtol=1e-5)
    assert tr.changed[0] == w.n
    assert st["certified"] >= 0.9 * w.n * iters


def test_hd_convergence_and_determinism():
    P, C0 = synth.random_instance(14, 8000, 128, 20, "blobs")
    a = run(P, C0, 100, tol=0.0)
    b = run(P, C0, 100, tol=0.0)
    assert a[0] < 100 and a[0] == b[0]
    np.testing.assert_array_equal(a[3], b[3])
    np.testing.assert_array_equal(a[2], b[2])
    r = oracle.lloyd(P, C0.astype(np.float64), 100, 0.0, True)
    assert a[0] == r.iterations
    np.testing.assert_array_equal(a[3], r.labels)


@pytest.mark.parametrize("cfg", [6, 7])
def test_hd_full_size_sampled(cfg):
    """Configs 6 / 7 at full size (n = 5e5, d = 128 / 256, k = 1000) in bench.py's launch
    configuration: labels of iteration 2 on a seeded sample against the oracle given the
    GPU's C_1; the refine of iteration 2 recomputed by the oracle over all n."""
    w = synth.config(cfg)
    ctx = kmb.Context(w.n, w.d, w.k)
    Pd = T(w.points)
    _, _, C1, _, _ = run_ctx(ctx, Pd, w.init, 1)
    it, sse, C2, lab2, tr = run_ctx(ctx, Pd, w.init, 2)
    ctx.close()
    s = np.random.default_rng(0).choice(w.n, 4000, replace=False)
    a = oracle.assign(w.points[s], C1.astype(np.float64))
    np.testing.assert_array_equal(lab2[s], a.labels)
    u = oracle.update(w.points, lab2, C1.astype(np.float64), round_f32=True)
    assert_centroids_close(C2, u.centroids, w.points)
    assert_sse_close(sse, oracle.sse(w.points, lab2, C2.astype(np.float64)))


@pytest.mark.parametrize("d,k,kind", [(128, 3, "blobs"), (256, 300, "blobs"), (64, 40, "grid")])
def test_hd_forced_fallback(d, k, kind):
    """km_debug_set(KM_DBG_HD, 4) sends every point to the FP64 fallback (the sliced pair for the first 4096,
    8 points per CTA over all k for the rest; reduce-scattered partial sums, sequential FP64 on
    near-ties): labels must still be the oracle's."""
    n = 6000   # > kFbCap (4096): both the sliced pair and the all-k kernel run
    P, C0 = synth.random_instance(15 + d, n, d, k, kind)
    st = lockstep(P, C0, 2, hd_dbg=4)
    assert st["full_scan"] == n and st["certified"] == 0   # (stats of the last one-iteration run)


@pytest.mark.parametrize("d", [64, 256])
def test_hd_assign_update_abi(d):
    """The per-step ABI (km_assign, km_update) at high d, lockstep with the oracle: labels
    identical, SSE_t, counts, centroids and drift within the parity tolerance."""
    n, k = 3001, 40
    P, C0 = synth.random_instance(21 + d, n, d, k, "blobs")
    ctx = kmb.Context(n, d, k)
    Pd = T(P)
    C = C0.astype(np.float64)
    for t in range(3):
        lab = torch.empty(n, dtype=torch.int32, device=dev)
        sse = torch.zeros(1, dtype=torch.float64, device=dev)
        kmb.km_assign(ctx.handle, Pd, T(C.astype(np.float32)), lab, sse)
        torch.cuda.synchronize()
        a = oracle.assign(P, C)
        np.testing.assert_array_equal(lab.cpu().numpy(), a.labels, err_msg=f"step {t}")
        assert_sse_close(float(sse.item()), a.best.sum(), rel=1e-9)
        new = torch.empty((k, d), dtype=torch.float32, device=dev)
        cnt = torch.empty(k, dtype=torch.int32, device=dev)
        md = torch.zeros(1, dtype=torch.float64, device=dev)
        kmb.km_update(ctx.handle, Pd, lab, T(C.astype(np.float32)), new, cnt, md)
        torch.cuda.synchronize()
        u = oracle.update(P, a.labels, C, round_f32=True)
        np.testing.assert_array_equal(cnt.cpu().numpy(), u.counts)
        assert_centroids_close(new.cpu().numpy(), u.centroids, P)
        assert abs(float(md.item()) - u.max_drift) <= 1e-4 * max(u.max_drift, 1e-3) + 1e-12
        C = u.centroids
    ctx.close()


def test_hd_top8_large_k():
    """k > 2048 keeps the top 8 per column half (crowded bands at large k): lockstep labels,
    plus 12 copies of one centroid (more than 8 in the band -> the FP64 scan over all k)."""
    P, C0 = synth.random_instance(31, 8000, 64, 2600, "blobs")
    C0 = C0.copy()
    C0[2000:2012] = C0[5]
    lockstep(P, C0, 2)


def test_hd_identical_points_and_centroids():
    """Degenerate: every point identical, every centroid identical (zero box extent, all scores
    tie exactly): all labels 0 (lowest index), SSE 0, centroid 0 = the point, others kept."""
    n, d, k = 1000, 128, 5
    P = np.tile(np.linspace(-3, 3, d, dtype=np.float32), (n, 1))
    C0 = P[:k].copy()
    it, sse, C, lab, tr, st = run(P, C0, 3)
    assert (lab == 0).all() and sse == 0.0
    np.testing.assert_array_equal(C, C0)
    a = oracle.assign(P, C0.astype(np.float64))
    assert (a.labels == 0).all()


@pytest.mark.parametrize("d,n,k", [(4, 3001, 37), (17, 2000, 20), (100, 5000, 300), (200, 3001, 64)])
def test_hd_padded_width_lockstep(d, n, k):
    """d outside {2, 3, 32, 64, 128, 256} runs on points zero-padded to the next native width:
    labels identical to the oracle on the unpadded data, centroids come back [k][d]."""
    P, C0 = synth.random_instance(5 * n + d + k, n, d, k, "blobs")
    lockstep(P, C0, 3)


@pytest.mark.parametrize("d", [24, 130])
def test_hd_padded_width_abi_and_host(d):
    """Padded widths through km_assign / km_update (device) and km_run (host arrays), against the
    oracle; km_update may update in place."""
    n, k = 2500, 30
    P, C0 = synth.random_instance(77 + d, n, d, k, "blobs")
    ctx = kmb.Context(n, d, k)
    Pd = T(P)
    lab = torch.empty(n, dtype=torch.int32, device=dev)
    sse = torch.zeros(1, dtype=torch.float64, device=dev)
    Cd = T(C0.astype(np.float32))
    kmb.km_assign(ctx.handle, Pd, Cd, lab, sse)
    torch.cuda.synchronize()
    a = oracle.assign(P, C0.astype(np.float64))
    np.testing.assert_array_equal(lab.cpu().numpy(), a.labels)
    assert_sse_close(float(sse.item()), a.best.sum(), rel=1e-9)
    cnt = torch.empty(k, dtype=torch.int32, device=dev)
    kmb.km_update(ctx.handle, Pd, lab, Cd, Cd, cnt, None)
    torch.cuda.synchronize()
    u = oracle.update(P, a.labels, C0.astype(np.float64), round_f32=True)
    np.testing.assert_array_equal(cnt.cpu().numpy(), u.counts)
    assert_centroids_close(Cd.cpu().numpy(), u.centroids, P)
    ctx.close()
    Ch = np.empty((k, d), np.float32)
    lh = np.empty(n, np.int32)
    it, sse_h = kmb.km_run(P, n, d, k, C0, 4, -1.0, Ch, lh)
    r = oracle.lloyd(P, C0.astype(np.float64), 4, tol=-1.0)
    assert it == 4
    np.testing.assert_array_equal(lh, r.labels)
    assert_centroids_close(Ch, r.centroids, P)


def test_hd_host_pointers_and_km_run():
    """km_run (the north-star call) with host arrays, against km_run_ctx on device buffers."""
    w = synth.config(6, n=9000, k=50)
    n, d, k = w.n, w.d, w.k
    Cd = np.empty((k, d), np.float32)
    ld = np.empty(n, np.int32)
    it, sse = kmb.km_run(w.points, n, d, k, w.init, 4, -1.0, Cd, ld)
    it2, sse2, C2, l2, _, _ = run(w.points, w.init, 4)
    assert it == it2 == 4 and sse == sse2
    np.testing.assert_array_equal(Cd, C2)
    np.testing.assert_array_equal(ld, l2)
