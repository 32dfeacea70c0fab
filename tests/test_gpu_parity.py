"""GPU parity: libkm (through the C ABI) against the FP64 oracle, element by element.

Lockstep (the gate): both sides use the oracle's float32 centroids C_t each
iteration; labels must be IDENTICAL, SSE_t and the update within tolerance.
Free run: km_run vs oracle.lloyd (mode A) from the same C0.
Full-size configs run in bench.py's launch configuration and are checked on
sampled outputs (labels of a seeded sample recomputed by the oracle) plus exact
O(nd) recomputations (update, Eq. 1).
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


def T(a, dtype=None):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def gpu_assign(ctx, Pd, C):
    lab = torch.empty(Pd.shape[0], dtype=torch.int32, device=dev)
    sse = torch.zeros(1, dtype=torch.float64, device=dev)
    kmb.km_assign(ctx.handle, Pd, T(np.asarray(C, np.float32)), lab, sse)
    torch.cuda.synchronize()
    return lab.cpu().numpy(), float(sse.item())


def gpu_update(ctx, Pd, lab, C):
    k, d = C.shape
    new = torch.empty((k, d), dtype=torch.float32, device=dev)
    cnt = torch.empty(k, dtype=torch.int32, device=dev)
    md = torch.zeros(1, dtype=torch.float64, device=dev)
    kmb.km_update(ctx.handle, Pd, T(np.asarray(lab, np.int32)), T(np.asarray(C, np.float32)), new, cnt, md)
    torch.cuda.synchronize()
    return new.cpu().numpy(), cnt.cpu().numpy(), float(md.item())


def gpu_run(P, C0, iters, tol=-1.0, variant=None):
    n, d = P.shape
    k = C0.shape[0]
    ctx = kmb.Context(n, d, k)
    if variant is not None:
        kmlib.km_debug_set_variant(ctx.handle, variant)
    Pd, C0d = T(P), T(C0)
    Cout = torch.empty((k, d), dtype=torch.float32, device=dev)
    lab = torch.empty(n, dtype=torch.int32, device=dev)
    it, sse = kmb.km_run_ctx(ctx.handle, Pd, C0d, iters, tol, Cout, lab)
    tr = kmb.km_read_traces(ctx.handle, iters)
    ctx.close()
    return it, sse, Cout.cpu().numpy(), lab.cpu().numpy(), tr


def lockstep(P, C0, iters, variant=None, check_counts=True):
    n, d = P.shape
    k = C0.shape[0]
    ctx = kmb.Context(n, d, k)
    if variant is not None:
        kmlib.km_debug_set_variant(ctx.handle, variant)
    Pd = T(P)
    C = C0.astype(np.float64)
    mism = 0
    for t in range(iters):
        lab_g, sse_g = gpu_assign(ctx, Pd, C)
        a = oracle.assign(P, C)
        np.testing.assert_array_equal(lab_g, a.labels, err_msg=f"iteration {t}: labels differ")
        assert_sse_close(sse_g, a.best.sum(), rel=1e-12)
        Cg, cnt_g, md_g = gpu_update(ctx, Pd, lab_g, C)
        u = oracle.update(P, a.labels, C, round_f32=True)
        if check_counts:
            np.testing.assert_array_equal(cnt_g, u.counts)
        mism += assert_centroids_close(Cg, u.centroids, P)
        assert abs(md_g - u.max_drift) <= 1e-4 * max(u.max_drift, 1e-3 * max(1.0, np.abs(C).max())) + 1e-12
        C = u.centroids
    ctx.close()
    return mism


# ------------------------------------------------------------------ hand examples
def test_gpu_hand_examples():
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hand_examples.json")))
    for case in g["lloyd"]:
        if case.get("grid10"):
            P = np.array([[x, y] for x in range(10) for y in range(10)], np.float32)
        else:
            P = np.array(case["points"], np.float32)
        if P.shape[1] == 1:   # embed the 1-D example in 2-D (y = 0)
            P = np.concatenate([P, np.zeros_like(P)], 1)
            C0 = np.concatenate([np.array(case["init"], np.float32), np.zeros((len(case["init"]), 1), np.float32)], 1)
        else:
            C0 = np.array(case["init"], np.float32)
        it, sse, C, lab, tr = gpu_run(P, C0, 20, tol=float(case["tol"]))
        assert it == case["iterations"]
        want = [[float(v[0]) / v[1] for v in c] for c in case["centroids"]]
        np.testing.assert_array_equal(C[:, :len(want[0])], np.array(want, np.float32))
        if "labels" in case:
            assert lab.tolist() == case["labels"]
        ws = case["out_sse"]
        assert sse == ws[0] / ws[1]
        wt = [v[0] / v[1] for v in case["sse_trace"]]
        np.testing.assert_allclose(tr.sse, wt, rtol=1e-6)
        if "changed_trace" in case:
            assert tr.changed.tolist() == case["changed_trace"]


def test_gpu_assign_hand_cases():
    g = __import__("json").load(open(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden",
                                                                "hand_examples.json")))
    for case in g["assign"]:
        P = np.array(case["points"], np.float32)
        C = np.array(case["centroids"], np.float32)
        if len(C) > len(P):   # k <= n: replicate the point
            P = np.repeat(P, len(C), 0)
        ctx = kmb.Context(len(P), P.shape[1], len(C))
        lab, sse = gpu_assign(ctx, T(P), C)
        assert (lab == case["labels"][0]).all(), case["cite"]
        assert sse == case["best"][0] * len(P)
        ctx.close()


# ------------------------------------------------------------------ lockstep on configs
@pytest.mark.parametrize("variant", list(range(9)))
def test_lockstep_config1(variant):
    w = synth.config(1)
    lockstep(w.points, w.init, w.iters, variant)


@pytest.mark.parametrize("variant", list(range(9)))
def test_lockstep_config2(variant):
    w = synth.config(2)
    lockstep(w.points, w.init, 8 if variant == 0 else w.iters, variant)


@pytest.mark.parametrize("variant", [1, 2])
def test_lockstep_config3_full_n(variant):
    w = synth.config(3)
    lockstep(w.points, w.init, 3, variant)


def test_lockstep_config4_shape_small_n():
    w = synth.config(4, n=200_000, k=1000)
    lockstep(w.points, w.init, 4)


# ------------------------------------------------------------------ free runs
@pytest.mark.parametrize("cfg,n", [(1, None), (2, None), (3, 100_000)])
def test_free_run_configs(cfg, n):
    w = synth.config(cfg, n=n)
    it, sse, C, lab, tr = gpu_run(w.points, w.init, w.iters)
    assert it == w.iters
    r = oracle.lloyd(w.points, w.init.astype(np.float64), w.iters, -1.0, True)
    rp = oracle.lloyd(w.points, w.init.astype(np.float64), w.iters - 1, -1.0, True)
    assert_centroids_close(C, r.centroids, w.points)
    assert_sse_close(sse, r.sse)
    assert_labels_near_tie_only(w.points, lab, rp.centroids)
    np.testing.assert_allclose(tr.sse, r.sse_trace, rtol=1e-5)
    assert tr.changed[0] == w.n


@pytest.mark.parametrize("seed", range(40))
def test_random_instances_free_run(seed):
    """SPEC-style harness: seeded instances n <= 2000, k <= 32, d in {2,3}."""
    rng = np.random.default_rng(seed)
    d = 2 + seed % 2
    n = int(rng.integers(40, 2000))
    k = int(rng.integers(1, 33))
    kind = ["blobs", "uniform", "grid", "offset"][seed % 4]
    P, C0 = synth.random_instance(1000 + seed, n, d, k, kind)
    iters = 12
    it, sse, C, lab, tr = gpu_run(P, C0, iters)
    r = oracle.lloyd(P, C0.astype(np.float64), iters, -1.0, True)
    rp = oracle.lloyd(P, C0.astype(np.float64), iters - 1, -1.0, True)
    assert_centroids_close(C, r.centroids, P)
    assert_sse_close(sse, r.sse)
    assert_labels_near_tie_only(P, lab, rp.centroids)


# ------------------------------------------------------------------ edge cases
@pytest.mark.parametrize("n", [1, 3, 31, 33, 255, 257, 1023, 1025, 10_007])
@pytest.mark.parametrize("d", [2, 3])
def test_tails(n, d):
    k = min(n, 7)
    P, C0 = synth.random_instance(n + d, n, d, k, "blobs")
    lockstep(P, C0, 3)


def test_k1_and_k_equals_n():
    P, _ = synth.random_instance(5, 3000, 3, 1, "uniform")
    it, sse, C, lab, tr = gpu_run(P, P[:1].copy(), 3)
    assert (lab == 0).all()
    np.testing.assert_allclose(C[0], P.astype(np.float64).mean(0), rtol=1e-6)
    Q, _ = synth.random_instance(6, 500, 2, 1, "uniform")
    it, sse, C, lab, tr = gpu_run(Q, Q.copy(), 5, tol=0.0)
    assert it == 1 and sse == 0.0
    assert lab.tolist() == list(range(500))


def test_duplicate_centroids_and_ties():
    # integer lattice: many exact FP32/FP64 ties; duplicated centroids: lower index wins
    P, C0 = synth.random_instance(7, 5000, 2, 16, "grid")
    C0 = C0.copy()
    C0[5] = C0[3]
    C0[9] = C0[3]
    mism = lockstep(P, C0, 5)
    lab, _ = gpu_assign(kmb.Context(len(P), 2, 16), T(P), C0.astype(np.float64))
    assert not ((lab == 5) | (lab == 9)).any()


def test_all_points_identical():
    P = np.full((1000, 3), 2.5, np.float32)
    C0 = np.array([[2.5, 2.5, 2.5], [0, 0, 0]], np.float32)
    it, sse, C, lab, tr = gpu_run(P, C0, 4, tol=0.0)
    assert (lab == 0).all() and sse == 0.0
    np.testing.assert_array_equal(C, C0)   # cluster 1 empty: kept (R5)


def test_offset_data_and_empty_clusters():
    P, C0 = synth.random_instance(8, 20_000, 2, 50, "offset")
    C0 = C0.copy()
    C0[:5] += 1000.0   # far centroids: stay empty forever
    lockstep(P, C0, 5)


def test_max_k():
    for d in (2, 3):
        kmax = kmb.km_max_k(d)
        n = kmax + 3000
        P, C0 = synth.random_instance(9 + d, n, d, kmax, "uniform")
        ctx = kmb.Context(n, d, kmax)
        lab, sse = gpu_assign(ctx, T(P), C0)
        idx = np.random.default_rng(0).choice(n, 2000, replace=False)
        a = oracle.assign(P[idx], C0.astype(np.float64))
        np.testing.assert_array_equal(lab[idx], a.labels)
        ctx.close()
        with pytest.raises(kmb.KmError):
            kmb.Context(n + 10, d, kmax + 1)


def test_host_pointers_and_km_run():
    w = synth.config(2, n=50_000)
    n, d, k = w.n, w.d, w.k
    Cd = np.empty((k, d), np.float32)
    ld = np.empty(n, np.int32)
    it, sse = kmb.km_run(w.points, n, d, k, w.init, 6, -1.0, Cd, ld)   # host in, host out
    it2, sse2, C2, l2, _ = gpu_run(w.points, w.init, 6)                 # device in/out via ctx
    assert it == it2 == 6 and sse == sse2
    np.testing.assert_array_equal(Cd, C2)
    np.testing.assert_array_equal(ld, l2)
    # pinned host buffers
    Pp = torch.from_numpy(w.points).pin_memory()
    Cp = torch.empty((k, d), dtype=torch.float32).pin_memory()
    lp = torch.empty(n, dtype=torch.int32).pin_memory()
    ctx = kmb.Context(n, d, k)
    it3, sse3 = kmb.km_run_ctx(ctx.handle, Pp, torch.from_numpy(w.init), 6, -1.0, Cp, lp)
    assert sse3 == sse
    np.testing.assert_array_equal(Cp.numpy(), Cd)
    ctx.close()


def test_convergence_and_determinism():
    w = synth.config(2, n=100_000)
    r = oracle.lloyd(w.points, w.init.astype(np.float64), 300, 0.0, True)
    it, sse, C, lab, tr = gpu_run(w.points, w.init, 300, tol=0.0)
    assert it == r.iterations
    np.testing.assert_array_equal(lab, r.labels)
    assert_centroids_close(C, r.centroids, w.points)
    it2, sse2, C2, lab2, tr2 = gpu_run(w.points, w.init, 300, tol=0.0)
    assert it2 == it and sse2 == sse
    np.testing.assert_array_equal(C2, C)
    np.testing.assert_array_equal(lab2, lab)
    np.testing.assert_array_equal(tr2.sse, tr.sse)


def test_variants_agree_bitwise():
    w = synth.config(3, n=300_000)
    a = gpu_run(w.points, w.init, 5, variant=0)
    for v in range(1, 7):
        b = gpu_run(w.points, w.init, 5, variant=v)
        np.testing.assert_array_equal(a[3], b[3])
        np.testing.assert_array_equal(a[2], b[2])
        assert a[1] == b[1]


# ------------------------------------------------------------------ full-size configs (bench launch config)
@pytest.mark.parametrize("cfg", [4, 5])
def test_full_size_sampled(cfg):
    w = synth.config(cfg)
    T_ = w.iters
    itp, _, Cprev, _, _ = gpu_run(w.points, w.init, T_ - 1)
    it, sse, C, lab, tr = gpu_run(w.points, w.init, T_)
    assert it == T_ and itp == T_ - 1
    # labels of a seeded sample recomputed by the oracle against C_{T-1}: exact
    idx = np.random.default_rng(cfg).choice(w.n, 20_000, replace=False)
    a = oracle.assign(w.points[idx], Cprev.astype(np.float64))
    np.testing.assert_array_equal(lab[idx], a.labels)
    # C_T is the exact refine of (labels, C_{T-1})
    u = oracle.update(w.points, lab, Cprev.astype(np.float64), round_f32=True)
    assert_centroids_close(C, u.centroids, w.points)
    # out_sse is Eq. 1 of the returned pair
    assert_sse_close(sse, oracle.sse(w.points, lab, C.astype(np.float64)))
    # SSE_t non-increasing (mode-A slack)
    assert (np.diff(tr.sse) <= 1e-6 * tr.sse[:-1]).all()


# ------------------------------------------------------------- A6: CUDA-graph replay
def _run_ctx(ctx, Pd, C0d, iters, tol):
    k, d = C0d.shape
    Cout = torch.empty((k, d), dtype=torch.float32, device=dev)
    lab = torch.empty(Pd.shape[0], dtype=torch.int32, device=dev)
    st = torch.zeros(iters, dtype=torch.float64, device=dev)
    ct = torch.zeros(iters, dtype=torch.int64, device=dev)
    it, sse = kmb.km_run_ctx(ctx.handle, Pd, C0d, iters, tol, Cout, lab, st, ct)
    tr = kmb.km_read_traces(ctx.handle, iters)
    return it, sse, Cout.cpu().numpy(), lab.cpu().numpy(), st.cpu().numpy(), ct.cpu().numpy(), tr.max_drift


@pytest.mark.parametrize("cfg,n,k,mode", [(1, None, None, kmb.KM_MODE_AUTO), (2, 200_000, None, kmb.KM_MODE_AUTO),
                                          (3, 100_000, None, kmb.KM_MODE_TILES),
                                          (3, 100_000, None, kmb.KM_MODE_BRUTE)])
@pytest.mark.parametrize("tol", [-1.0, 0.0])
def test_graph_replay_equals_eager(cfg, n, k, mode, tol):
    """km_run_ctx captures its device work once as a CUDA graph (loop control of Alg. 1,
    P:L286) and replays it; replays must equal eager launches bit for bit, pick up
    new data written into the same buffers, and stop on the device flag when tol >= 0."""
    w = synth.config(cfg, n=n, k=k)
    iters = w.iters
    ctx_e = kmb.Context(w.n, w.d, w.k)
    kmb.km_set_mode(ctx_e.handle, mode)
    kmlib.km_debug_set(ctx_e.handle, kmlib.KM_DBG_GRAPH, 0)
    ctx_g = kmb.Context(w.n, w.d, w.k)
    kmb.km_set_mode(ctx_g.handle, mode)
    Pd, C0d = T(w.points), T(w.init)
    ref = _run_ctx(ctx_e, Pd, C0d, iters, tol)
    l0 = kmb.km_launch_count(ctx_g.handle, reset=True)
    for rep in range(3):   # capture, then two replays
        got = _run_ctx(ctx_g, Pd, C0d, iters, tol)
        assert got[0] == ref[0]
        assert got[1] == ref[1]
        for a, b in zip(got[2:], ref[2:]):
            np.testing.assert_array_equal(a, b)
    assert kmb.km_launch_count(ctx_g.handle) > l0
    if tol >= 0 and ref[0] < iters:   # unexecuted iterations: NaN / -1
        assert np.isnan(got[4][ref[0]:]).all() and (got[5][ref[0]:] == -1).all()
    # new data in the same buffers: the replay must compute on it
    rng = np.random.default_rng(5)
    P2 = (w.points + rng.normal(0, 0.01, w.points.shape)).astype(np.float32)
    Pd.copy_(T(P2))
    got2 = _run_ctx(ctx_g, Pd, C0d, iters, tol)
    ref2 = _run_ctx(ctx_e, Pd, C0d, iters, tol)
    assert got2[0] == ref2[0] and got2[1] == ref2[1]
    np.testing.assert_array_equal(got2[3], ref2[3])
    np.testing.assert_array_equal(got2[2], ref2[2])
    ctx_e.close()
    ctx_g.close()


def test_privatised_update_near_zero_cluster_in_wide_box():
    """the fixed-point quantum is absolute (2^-s_m, s_m from n and the box extent):
    a cluster near 0 inside a wide box gets centroids within 2^-(s_m+1) of the FP64 mean plus
    the float32 rounding -- checked against the oracle with that bound (km.h km_run_ctx)."""
    rng = np.random.default_rng(8)
    n = 50_000
    P = np.concatenate([rng.normal(0, 1e-4, (n // 2, 2)), rng.uniform(-1000, 1000, (n - n // 2, 2))]).astype(np.float32)
    P = P[rng.permutation(n)]
    C0 = np.concatenate([[[0.0, 0.0]], P[rng.choice(n, 15, replace=False)]]).astype(np.float32)
    ctx = kmb.Context(n, 2, 16)
    Pd = T(P)
    lab, _ = gpu_assign(ctx, Pd, C0.astype(np.float64))
    Cg, cnt, _ = gpu_update(ctx, Pd, lab, C0.astype(np.float64))
    ctx.close()
    u = oracle.update(P, lab, C0.astype(np.float64), round_f32=True)
    np.testing.assert_array_equal(cnt, u.counts)
    ext = (P.max(0).astype(np.float64) - P.min(0))
    nb = int(n).bit_length()
    s = 61 - nb - np.frexp(ext)[1]
    bound = 2.0 ** -(s + 1) + np.spacing(np.abs(u.centroids).astype(np.float32)).astype(np.float64)
    assert (np.abs(Cg - u.centroids) <= bound).all()
    assert abs(Cg[0]).max() < 1e-3   # the near-zero cluster stays near zero


@pytest.mark.parametrize("seed,n,d,k,kind,tol", [(1, 10_000, 2, 10, "uniform", -1.0), (2, 65_536, 3, 1000, "blobs", -1.0),
                                                 (3, 777, 2, 37, "grid", 0.0), (4, 40_000, 3, 64, "offset", 0.0),
                                                 (5, 5, 2, 5, "blobs", -1.0)])
def test_small_run_kernel_equals_multi_kernel(seed, n, d, k, kind, tol):
    """Brute-force runs with n <= 65536 execute as one launch of one CTA (km_small.cuh): labels,
    centroids, iterations, changed_t, drift and out_sse equal the multi-kernel sequence bit for
    bit (SSE_t up to FP64 summation order), and the labels the oracle's."""
    P, C0 = synth.random_instance(600 + seed, n, d, k, kind)
    outs = []
    for small in (1, 0):
        ctx = kmb.Context(n, d, k)
        kmb.km_set_mode(ctx.handle, kmb.KM_MODE_BRUTE)
        kmlib.km_debug_set(ctx.handle, kmlib.KM_DBG_SMALL, small)
        outs.append(_run_ctx(ctx, T(P), T(C0), 15, tol))
        ctx.close()
    a, b = outs
    assert a[0] == b[0] and a[1] == b[1]
    np.testing.assert_array_equal(a[2], b[2])
    np.testing.assert_array_equal(a[3], b[3])
    np.testing.assert_array_equal(a[5], b[5])
    np.testing.assert_array_equal(a[6][:a[0]], b[6][:b[0]])
    np.testing.assert_allclose(a[4][:a[0]], b[4][:b[0]], rtol=1e-12)
    r = oracle.lloyd(P, C0.astype(np.float64), 15, tol, True)
    assert r.iterations == a[0]
    np.testing.assert_array_equal(a[3], r.labels)
    assert_sse_close(a[1], r.sse, rel=1e-12)
