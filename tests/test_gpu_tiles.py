"""GPU parity of the tile-pruned path (KM_MODE_TILES, the paper's batch assignment).

Pruning must never change the result: labels are certified against FP64
and sums are exact integers, so TILES must reproduce BRUTE bit for bit (labels,
centroids, iteration count, changed trace) and match the FP64 oracle.
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


def run(P, C0, iters, mode, tol=-1.0, dbg=None):
    n, d = P.shape
    k = C0.shape[0]
    ctx = kmb.Context(n, d, k)
    kmb.km_set_mode(ctx.handle, mode)
    for what, value in (dbg or {}).items():
        kmlib.km_debug_set(ctx.handle, what, value)
    Pd = torch.from_numpy(P).to(dev)
    C0d = torch.from_numpy(np.ascontiguousarray(C0)).to(dev)
    Cout = torch.empty((k, d), dtype=torch.float32, device=dev)
    lab = torch.empty(n, dtype=torch.int32, device=dev)
    it, sse = kmb.km_run_ctx(ctx.handle, Pd, C0d, iters, tol, Cout, lab)
    tr = kmb.km_read_traces(ctx.handle, iters)
    st = kmb.km_read_stats(ctx.handle)
    ctx.close()
    return dict(it=it, sse=sse, C=Cout.cpu().numpy(), lab=lab.cpu().numpy(), tr=tr, st=st)


def same(a, b):
    assert a["it"] == b["it"]
    np.testing.assert_array_equal(a["lab"], b["lab"])
    np.testing.assert_array_equal(a["C"], b["C"])
    np.testing.assert_array_equal(a["tr"].changed, b["tr"].changed)
    np.testing.assert_array_equal(a["tr"].max_drift, b["tr"].max_drift)
    # SSE_t: the tile path sums certified FP32 distances / tile moments: within 1e-6
    np.testing.assert_allclose(a["tr"].sse, b["tr"].sse, rtol=2e-6)
    assert abs(a["sse"] - b["sse"]) <= 1e-12 * max(abs(b["sse"]), 1e-300)


@pytest.mark.parametrize("cfg,n,k,iters", [(1, 50_000, 10, 10), (2, None, None, 20), (3, None, None, 8),
                                           (4, 2_000_000, None, 6), (5, 2_000_000, 2000, 4)])
def test_tiles_equal_brute(cfg, n, k, iters):
    w = synth.config(cfg, n=n, k=k)
    a = run(w.points, w.init, iters, kmb.KM_MODE_TILES)
    b = run(w.points, w.init, iters, kmb.KM_MODE_BRUTE)
    same(a, b)
    assert a["st"]["tiles"] and a["st"]["pairs"] < b["st"]["pairs"]


def test_tiles_vs_oracle_config3_sample():
    w = synth.config(3, n=200_000)
    a = run(w.points, w.init, 10, kmb.KM_MODE_TILES)
    r = oracle.lloyd(w.points, w.init.astype(np.float64), 10, -1.0, True)
    rp = oracle.lloyd(w.points, w.init.astype(np.float64), 9, -1.0, True)
    assert_centroids_close(a["C"], r.centroids, w.points)
    assert_sse_close(a["sse"], r.sse)
    assert_labels_near_tie_only(w.points, a["lab"], rp.centroids)
    np.testing.assert_allclose(a["tr"].sse, r.sse_trace, rtol=1e-5)


@pytest.mark.parametrize("n", [1, 1000, 1024, 1025, 4095, 16384 + 37])
@pytest.mark.parametrize("d", [2, 3])
def test_tiles_ragged(n, d):
    k = min(n, 9)
    P, C0 = synth.random_instance(n * 7 + d, n, d, k, "blobs")
    same(run(P, C0, 5, kmb.KM_MODE_TILES), run(P, C0, 5, kmb.KM_MODE_BRUTE))


@pytest.mark.parametrize("kind", ["grid", "offset", "uniform"])
def test_tiles_ties_offset(kind):
    P, C0 = synth.random_instance(77, 60_000, 2, 40, kind)
    C0 = C0.copy()
    C0[7] = C0[3]    # duplicate centroid: never a batch tile, lower index wins
    a = run(P, C0, 6, kmb.KM_MODE_TILES)
    same(a, run(P, C0, 6, kmb.KM_MODE_BRUTE))
    a1 = run(P, C0, 1, kmb.KM_MODE_TILES)    # first assignment: the twin (index 7) never wins
    assert not (a1["lab"] == 7).any()


def test_tiles_k1_identical_points_and_overflow():
    P, _ = synth.random_instance(3, 20_000, 3, 1, "uniform")
    a = run(P, P[:1].copy(), 3, kmb.KM_MODE_TILES)
    same(a, run(P, P[:1].copy(), 3, kmb.KM_MODE_BRUTE))
    assert a["st"]["batch_tiles"] == a["st"]["tile_visits"]      # k = 1: every tile in batch
    Q = np.full((5000, 2), 3.0, np.float32)
    C = np.array([[3, 3], [0, 0]], np.float32)
    same(run(Q, C, 3, kmb.KM_MODE_TILES, tol=0.0), run(Q, C, 3, kmb.KM_MODE_BRUTE, tol=0.0))
    # more candidates than the shared-memory list holds: the tile scans all k
    U, CU = synth.random_instance(5, 4096, 2, 3000, "uniform")
    same(run(U, CU, 3, kmb.KM_MODE_TILES), run(U, CU, 3, kmb.KM_MODE_BRUTE))


def test_tiles_convergence_tol0():
    w = synth.config(2, n=300_000)
    a = run(w.points, w.init, 300, kmb.KM_MODE_TILES, tol=0.0)
    same(a, run(w.points, w.init, 300, kmb.KM_MODE_BRUTE, tol=0.0))
    assert a["it"] < 300
    assert a["tr"].changed[-1] == 0 or a["tr"].max_drift[-1] == 0.0


def test_tiles_full_config4_sampled():
    """Headline workload in bench.py's launch configuration (AUTO -> tiles)."""
    w = synth.config(4)
    a = run(w.points, w.init, w.iters, kmb.KM_MODE_AUTO)
    assert a["st"]["tiles"]
    ap = run(w.points, w.init, w.iters - 1, kmb.KM_MODE_AUTO)
    idx = np.random.default_rng(4).choice(w.n, 20_000, replace=False)
    o = oracle.assign(w.points[idx], ap["C"].astype(np.float64))
    np.testing.assert_array_equal(a["lab"][idx], o.labels)
    u = oracle.update(w.points, a["lab"], ap["C"].astype(np.float64), round_f32=True)
    assert_centroids_close(a["C"], u.centroids, w.points)
    assert_sse_close(a["sse"], oracle.sse(w.points, a["lab"], a["C"].astype(np.float64)))


def test_tiles_edge_cases():
    """Single cluster, all points on one centroid, overflowing candidate lists, ragged tails."""
    P, _ = synth.random_instance(3, 20_000, 3, 1, "uniform")
    same(run(P, P[:1].copy(), 3, kmb.KM_MODE_TILES), run(P, P[:1].copy(), 3, kmb.KM_MODE_BRUTE))
    Q = np.full((5000, 2), 3.0, np.float32)
    C = np.array([[3, 3], [0, 0]], np.float32)
    same(run(Q, C, 3, kmb.KM_MODE_TILES, tol=0.0), run(Q, C, 3, kmb.KM_MODE_BRUTE, tol=0.0))
    U, CU = synth.random_instance(5, 4096, 2, 3000, "uniform")   # long candidate lists (overflow pool)
    same(run(U, CU, 3, kmb.KM_MODE_TILES), run(U, CU, 3, kmb.KM_MODE_BRUTE))
    for n in (16385, 20_000 + 77):   # ragged last tile (partly empty warps)
        R, CR = synth.random_instance(7, n, 2, 64, "blobs")
        same(run(R, CR, 6, kmb.KM_MODE_TILES), run(R, CR, 6, kmb.KM_MODE_BRUTE))


def test_tiles_split_subballs_exact():
    """Tiles whose Morton-consecutive points straddle a jump are pruned with two sub-balls
    (km_tiles.cuh TileSub): sparse uniform background + dense blobs (config 5's mix) makes such
    tiles; results stay bit-identical to brute force."""
    w = synth.config(5, n=1_500_000, k=3000)
    a = run(w.points, w.init, 4, kmb.KM_MODE_TILES)
    b = run(w.points, w.init, 4, kmb.KM_MODE_BRUTE)
    same(a, b)
    assert a["st"]["split_tiles"] > 0


def _fuzz_cases():
    rng = np.random.default_rng(2024)
    kinds = ["uniform", "blobs", "grid", "offset"]
    cases = []
    for i in range(32):
        d = int(rng.choice([2, 3]))
        n = int(rng.choice([1, 3, 127, 129, 16_384, 20_000, 65_537, 131_072, 300_001]))
        k = int(min(n, rng.choice([1, 2, 7, 64, 300, 1025, 2049, 3000])))
        cases.append((i, n, d, k, kinds[i % 4], int(rng.integers(2, 6))))
    return cases


@pytest.mark.parametrize("seed,n,d,k,kind,iters", _fuzz_cases())
def test_tiles_fuzz_equal_brute(seed, n, d, k, kind, iters):
    """Seeded random instances across sizes (ragged last tiles), k (flat index, hierarchical
    levels, CTA level-1 prune above 2048), distributions (lattice ties, offset data): the tile
    path equals brute force bit for bit."""
    P, C0 = synth.random_instance(100 + seed, n, d, k, kind)
    same(run(P, C0, iters, kmb.KM_MODE_TILES), run(P, C0, iters, kmb.KM_MODE_BRUTE))


@pytest.mark.parametrize("minb", [1, 2])
@pytest.mark.parametrize("cfg,n,k,iters", [(2, 300_000, None, 10), (3, 300_000, None, 6), (5, 1_500_000, 3000, 3)])
def test_tiles_k1t_register_variants_equal_brute(cfg, n, k, iters, minb):
    """K1t is built for two register budgets (MINB = 1: no spills, 8 warps/SM, chosen for few
    tiles; MINB = 2: 16 warps/SM, large problems); both must reproduce brute force bit for bit."""
    w = synth.config(cfg, n=n, k=k)
    a = run(w.points, w.init, iters, kmb.KM_MODE_TILES, dbg={kmlib.KM_DBG_K1T_MINB: minb})
    b = run(w.points, w.init, iters, kmb.KM_MODE_BRUTE)
    same(a, b)


@pytest.mark.parametrize("shift", [3, 4, 5])
@pytest.mark.parametrize("cfg,n,k,iters", [(2, 300_000, None, 10), (3, 300_000, None, 6), (4, 1_000_000, None, 4),
                                           (5, 1_500_000, 3000, 3)])
def test_tiles_super_tile_sizes_equal_brute(cfg, n, k, iters, shift):
    """Level-1 nodes of 8 tiles (chosen in 3-D), 16 (2-D) and 32 (2-D, k >= 4096): every index
    shape must reproduce brute force bit for bit in either dimension."""
    w = synth.config(cfg, n=n, k=k)
    a = run(w.points, w.init, iters, kmb.KM_MODE_TILES, dbg={kmlib.KM_DBG_ST_SHIFT: shift})
    b = run(w.points, w.init, iters, kmb.KM_MODE_BRUTE)
    same(a, b)


@pytest.mark.parametrize("short", [8, 48, 64])
@pytest.mark.parametrize("cfg,n,k,iters", [(3, 300_000, None, 6), (4, 1_000_000, None, 4), (5, 1_500_000, 3000, 3)])
def test_tiles_short_list_thresholds_equal_brute(cfg, n, k, iters, short):
    """The level-1 list length up to which the prune kernel expands the tiles' candidate lists
    itself (longer lists: one warp per tile, the multi-pass ones queued first) only moves work
    between two kernels: every threshold must reproduce brute force bit for bit."""
    w = synth.config(cfg, n=n, k=k)
    a = run(w.points, w.init, iters, kmb.KM_MODE_TILES, dbg={kmlib.KM_DBG_SHORT_LIST: short})
    b = run(w.points, w.init, iters, kmb.KM_MODE_BRUTE)
    same(a, b)


def test_tiles_label_scatter_multiwindow():
    """n above the label scatter's 12 M window (2 windows): the second window's labels come from
    the bucket the first pass fills; every label must land at its input position."""
    w = synth.config(5, n=13_000_000, k=256)
    a = run(w.points, w.init, 2, kmb.KM_MODE_TILES)
    b = run(w.points, w.init, 2, kmb.KM_MODE_BRUTE)
    same(a, b)
