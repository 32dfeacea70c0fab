"""GPU parity of KM_MODE_BOUNDS (brute force with per-point Hamerly bounds).

A point keeps its label without a scan only when its exact distance to its centroid (rounded
up) is below max(lb - dmax, s_a): the drift bound of P:L135 applied to the second-nearest
centroid and the inter bound of Eq. 4, both rounded down.  Such a skip never
changes a label, so BOUNDS must reproduce BRUTE bit for bit (labels, centroids, iteration
count, changed and drift traces, Eq. 1) and match the FP64 oracle -- while scanning far fewer
points.
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


def run(P, C0, iters, mode, tol=-1.0, dbg=None, graph=True):
    n, d = P.shape
    k = C0.shape[0]
    ctx = kmb.Context(n, d, k)
    kmb.km_set_mode(ctx.handle, mode)
    if not graph:
        kmlib.km_debug_set(ctx.handle, kmlib.KM_DBG_GRAPH, 0)
    for what, value in (dbg or {}).items():
        kmlib.km_debug_set(ctx.handle, what, value)
    Pd = torch.from_numpy(P).to(dev)
    C0d = torch.from_numpy(np.ascontiguousarray(C0)).to(dev)
    Cout = torch.empty((k, d), dtype=torch.float32, device=dev)
    lab = torch.empty(n, dtype=torch.int32, device=dev)
    it, sse = kmb.km_run_ctx(ctx.handle, Pd, C0d, iters, tol, Cout, lab)
    tr = kmb.km_read_traces(ctx.handle, iters)
    st = kmb.km_read_stats(ctx.handle)
    # a second call on the same context (graph replay, bounds re-initialised at t = 0)
    Cout2 = torch.empty_like(Cout)
    lab2 = torch.empty_like(lab)
    it2, sse2 = kmb.km_run_ctx(ctx.handle, Pd, C0d, iters, tol, Cout2, lab2)
    assert it2 == it and sse2 == sse
    assert torch.equal(Cout, Cout2) and torch.equal(lab, lab2)
    ctx.close()
    return dict(it=it, sse=sse, C=Cout.cpu().numpy(), lab=lab.cpu().numpy(), tr=tr, st=st)


def same(a, b):
    assert a["it"] == b["it"]
    np.testing.assert_array_equal(a["lab"], b["lab"])
    np.testing.assert_array_equal(a["C"], b["C"])
    np.testing.assert_array_equal(a["tr"].changed, b["tr"].changed)
    np.testing.assert_array_equal(a["tr"].max_drift, b["tr"].max_drift)
    # SSE_t: the same FP64 summands, summed per CTA in a different order
    np.testing.assert_allclose(a["tr"].sse, b["tr"].sse, rtol=1e-12)
    assert a["sse"] == b["sse"]   # Eq. 1 of the returned pair: 128-bit fixed point, order-free


@pytest.mark.parametrize("cfg,n,k,iters", [(2, None, None, 20), (1, 200_000, 10, 15), (3, 300_000, 200, 8),
                                           (3, 200_000, 700, 5), (5, 1_000_000, 64, 6)])
def test_bounds_equal_brute(cfg, n, k, iters):
    w = synth.config(cfg, n=n, k=k)
    a = run(w.points, w.init, iters, kmb.KM_MODE_BOUNDS)
    b = run(w.points, w.init, iters, kmb.KM_MODE_BRUTE)
    same(a, b)
    # the bounds skip work: fewer points scanned than n per iteration after the first
    assert a["st"]["points_scanned"] < b["st"]["points_scanned"]
    assert a["st"]["points_scanned"] >= w.n   # iteration 0 scans every point


@pytest.mark.parametrize("n", [1, 7, 2047, 2048, 2049, 70_001])
@pytest.mark.parametrize("d", [2, 3])
def test_bounds_ragged(n, d):
    k = min(n, 13)
    P, C0 = synth.random_instance(n * 5 + d, n, d, k, "blobs")
    same(run(P, C0, 6, kmb.KM_MODE_BOUNDS), run(P, C0, 6, kmb.KM_MODE_BRUTE))


@pytest.mark.parametrize("kind", ["grid", "offset", "uniform", "blobs"])
def test_bounds_ties_offset(kind):
    """Lattice points (exact distance ties: the lowest index wins, never by a skip), data far from
    the origin, a duplicated centroid (s_a = 0: its points are always scanned)."""
    P, C0 = synth.random_instance(91, 100_000, 2, 40, kind)
    C0 = C0.copy()
    C0[7] = C0[3]
    same(run(P, C0, 8, kmb.KM_MODE_BOUNDS), run(P, C0, 8, kmb.KM_MODE_BRUTE))


def test_bounds_convergence_and_eager():
    w = synth.config(2, n=300_000)
    a = run(w.points, w.init, 300, kmb.KM_MODE_BOUNDS, tol=0.0)
    same(a, run(w.points, w.init, 300, kmb.KM_MODE_BRUTE, tol=0.0))
    assert a["it"] < 300
    same(a, run(w.points, w.init, 300, kmb.KM_MODE_BOUNDS, tol=0.0, graph=False))


def test_bounds_vs_oracle_config2_lockstep():
    """Config 2 (the workload AUTO runs with bounds) against the FP64 oracle: labels of every
    iteration's final assignment, centroids, SSE_t trace, Eq. 1."""
    w = synth.config(2, n=250_000)
    a = run(w.points, w.init, 12, kmb.KM_MODE_BOUNDS)
    r = oracle.lloyd(w.points, w.init.astype(np.float64), 12, -1.0, True)
    rp = oracle.lloyd(w.points, w.init.astype(np.float64), 11, -1.0, True)
    assert_centroids_close(a["C"], r.centroids, w.points)
    assert_sse_close(a["sse"], r.sse)
    assert_labels_near_tie_only(w.points, a["lab"], rp.centroids)
    np.testing.assert_allclose(a["tr"].sse, r.sse_trace, rtol=1e-5)
    np.testing.assert_array_equal(a["tr"].changed, r.changed_trace)


def test_auto_picks_bounds_for_config2():
    w = synth.config(2, n=200_000)
    ctx = kmb.Context(w.n, w.d, w.k)
    P = torch.from_numpy(w.points).to(dev)
    C0 = torch.from_numpy(w.init).to(dev)
    C = torch.empty_like(C0)
    lab = torch.empty(w.n, dtype=torch.int32, device=dev)
    kmb.km_run_ctx(ctx.handle, P, C0, 8, -1.0, C, lab)
    st = kmb.km_read_stats(ctx.handle)
    ctx.close()
    assert not st["tiles"] and st["points_scanned"] < 8 * w.n


def test_bounds_pdl_off_equal():
    """Programmatic dependent launches between the iterations' kernels (default) change no result."""
    w = synth.config(2, n=400_000)
    a = run(w.points, w.init, 12, kmb.KM_MODE_BOUNDS)
    b = run(w.points, w.init, 12, kmb.KM_MODE_BOUNDS, dbg={kmlib.KM_DBG_PDL: 0})
    same(a, b)
