"""Pins for oracle/ (CPU only): the oracle is checked against things other than itself.

* hand-worked examples with exact rational answers (tests/golden/hand_examples.json,
  each case cites SPEC.md / SURVEY.md where the example comes from);
* exact rational arithmetic (oracle.pyref) on small integer instances;
* library special cases: scipy.cluster.vq.kmeans2 (mode B equals it: same
  assignment/empty-cluster/output conventions) and sklearn's KMeans on converged,
  well-separated data;
* closed forms (k = 1 -> mean and n*variance; k = n -> SSE 0) and invariants
  (argmin by brute force, sum of counts, SSE non-increasing, permutation
  equivariance, thread-count independence).
"""
import json
import os
import warnings
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import pyref
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hand_examples.json")))


def frac(v):
    return Fraction(v[0], v[1]) if isinstance(v, list) else Fraction(v)


def fr_arr(a):
    return np.array([[float(frac(x)) for x in row] for row in a])


def grid10():
    return np.array([[x, y] for x in range(10) for y in range(10)], np.float32)


# ---------------------------------------------------------------- hand examples
@pytest.mark.parametrize("case", GOLD["distance"], ids=lambda c: c["cite"][:20])
def test_distance_examples(case):
    P = np.array([case["p"]], np.float32)
    C = np.array([case["c"]], np.float64)
    r = oracle.assign(P, C)
    assert r.best[0] == case["sqdist"]
    assert pyref.sqdist(case["p"], case["c"]) == case["sqdist"]


@pytest.mark.parametrize("case", GOLD["assign"], ids=lambda c: c["cite"][:24])
def test_assign_examples(case):
    P = np.array(case["points"], np.float32)
    C = np.array(case["centroids"], np.float64)
    r = oracle.assign(P, C)
    assert r.labels.tolist() == case["labels"]
    assert r.best.tolist() == case["best"]
    assert r.second.tolist() == case["second"]
    lab, best = pyref.assign(case["points"], case["centroids"])
    assert lab == case["labels"] and best == case["best"]


@pytest.mark.parametrize("case", GOLD["update"], ids=lambda c: c["cite"][:24])
@pytest.mark.parametrize("mode_a", [True, False])
def test_update_examples(case, mode_a):
    P = np.array(case["points"], np.float32)
    r = oracle.update(P, case["labels"], np.array(case["old"], np.float64), round_f32=mode_a)
    np.testing.assert_array_equal(r.centroids, fr_arr(case["new"]))
    assert r.counts.tolist() == case["counts"]
    np.testing.assert_array_equal(r.drift, [float(frac(x)) for x in case["drift"]])
    assert r.max_drift == max(float(frac(x)) for x in case["drift"])


@pytest.mark.parametrize("case", GOLD["lloyd"], ids=lambda c: c["cite"][:24])
@pytest.mark.parametrize("mode_a", [True, False])
def test_lloyd_examples(case, mode_a):
    P = grid10() if case.get("grid10") else np.array(case["points"], np.float32)
    C0 = np.array(case["init"], np.float64)
    r = oracle.lloyd(P, C0, max_iter=20, tol=case["tol"], round_f32=mode_a)
    assert r.iterations == case["iterations"]
    want_c = fr_arr(case["centroids"])
    np.testing.assert_array_equal(r.centroids, want_c)   # final means are dyadic: exact in both modes
    if "labels" in case:
        assert r.labels.tolist() == case["labels"]
    if "changed_trace" in case:   # changed_0 counts every point (R6)
        assert r.changed_trace.tolist() == case["changed_trace"]
    want_trace = [float(frac(x)) for x in case["sse_trace"]]
    np.testing.assert_allclose(r.sse_trace, want_trace, rtol=1e-6 if mode_a else 1e-15)
    assert r.sse == float(frac(case["out_sse"]))
    # the exact-rational reference reproduces the same hand answers
    pts = P.astype(int).tolist() if case.get("grid10") else case["points"]
    C, lab, s, it, tr = pyref.lloyd(pts, case["init"], 20)
    assert it == case["iterations"] and s == frac(case["out_sse"])
    assert tr == [frac(x) for x in case["sse_trace"]]
    assert [[float(v) for v in c] for c in C] == want_c.tolist()
    if "labels0" in case:
        r1 = oracle.lloyd(P, C0, max_iter=1, tol=-1, round_f32=False)
        assert r1.labels.tolist() == case["labels0"]
        np.testing.assert_allclose(r1.centroids, fr_arr(case["centroids1"]), rtol=1e-15)


# ------------------------------------------------------- exact rational reference
@pytest.mark.parametrize("seed", range(12))
def test_against_exact_rationals(seed):
    """Integer data + integer-valued init: iteration 0 is exact in FP64, so labels,
    best distances and counts must equal the rational reference exactly; the whole
    mode-B run must match to FP64 rounding."""
    rng = np.random.default_rng(100 + seed)
    d = 2 + seed % 2
    n, k = 40 + seed, 2 + seed % 5
    P = rng.integers(-6, 7, (n, d)).astype(np.float32)
    C0 = P[rng.choice(n, k, replace=False)].astype(np.float64)
    r = oracle.assign(P, C0)
    lab, best = pyref.assign(P.astype(int).tolist(), C0.astype(int).tolist())
    assert r.labels.tolist() == lab
    assert r.best.tolist() == [float(b) for b in best]
    u = oracle.update(P, r.labels, C0, round_f32=False)
    Cx, cnt = pyref.update(P.astype(int).tolist(), lab, C0.astype(int).tolist())
    assert u.counts.tolist() == cnt
    np.testing.assert_allclose(u.centroids, [[float(v) for v in c] for c in Cx], rtol=1e-15, atol=0)
    # whole run: labels equal wherever the rational gap is not a near-tie
    res = oracle.lloyd(P, C0, max_iter=6, tol=-1, round_f32=False)
    C, lab_x, s_x, it, tr = pyref.lloyd(P.astype(int).tolist(), C0.astype(int).tolist(), 6, stop_at_fixpoint=False)
    assert it == 6
    assert res.labels.tolist() == lab_x
    np.testing.assert_allclose(res.sse_trace, [float(t) for t in tr], rtol=1e-13)
    np.testing.assert_allclose(res.sse, float(s_x), rtol=1e-13)


# ------------------------------------------------------------ library special case
def _kmeans2(P, C0, T):
    from scipy.cluster.vq import kmeans2
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return kmeans2(P.astype(np.float64), C0.astype(np.float64), iter=T, minit="matrix", missing="warn")


@pytest.mark.parametrize("seed,d,k,kind", [(0, 2, 5, "blobs"), (1, 3, 8, "blobs"), (2, 2, 16, "uniform"),
                                            (3, 3, 4, "grid"), (4, 2, 30, "blobs"), (5, 3, 12, "offset")])
def test_mode_b_equals_scipy_kmeans2(seed, d, k, kind):
    """scipy.cluster.vq.kmeans2(minit='matrix', iter=T) runs exactly T rounds of
    nearest-code assignment (lowest index on ties) + mean update keeping empty
    clusters, and returns (codebook after last update, last labels): mode B's
    conventions (R2, R3, R5)."""
    P, C0 = synth.random_instance(seed, 500, d, k, kind)
    T = 7
    cb, lab = _kmeans2(P, C0, T)
    r = oracle.lloyd(P, C0.astype(np.float64), max_iter=T, tol=-1, round_f32=False)
    assert r.iterations == T
    np.testing.assert_array_equal(r.labels, lab)
    np.testing.assert_allclose(r.centroids, cb, rtol=1e-12, atol=1e-12)


def test_mode_a_equals_kmeans2_rounded_each_iteration():
    """Mode A is kmeans2(iter=1) T times with the codebook rounded to float32 between calls."""
    P, C0 = synth.random_instance(7, 800, 3, 10, "blobs")
    C = C0.astype(np.float64)
    for _ in range(5):
        C, lab = _kmeans2(P, C, 1)
        C = C.astype(np.float32).astype(np.float64)
    r = oracle.lloyd(P, C0.astype(np.float64), max_iter=5, tol=-1, round_f32=True)
    np.testing.assert_array_equal(r.labels, lab)
    np.testing.assert_array_equal(r.centroids, C)


def test_sklearn_converged_well_separated():
    from sklearn.cluster import KMeans
    rng = np.random.default_rng(3)
    mu = np.array([[0, 0], [50, 0], [0, 50], [50, 50]], np.float64)
    P = (mu[rng.integers(0, 4, 2000)] + rng.normal(0, 1, (2000, 2))).astype(np.float32)
    C0 = np.array([P[np.argmin(np.linalg.norm(P - m, axis=1))] for m in mu], np.float64)
    r = oracle.lloyd(P, C0, max_iter=50, tol=0.0, round_f32=False)
    km = KMeans(4, init=C0, n_init=1, algorithm="lloyd", tol=0.0, max_iter=50).fit(P.astype(np.float64))
    np.testing.assert_array_equal(r.labels, km.labels_)
    np.testing.assert_allclose(r.centroids, km.cluster_centers_, rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(r.sse, km.inertia_, rtol=1e-10)


# ------------------------------------------------------- closed forms / invariants
def test_k1_is_mean_and_n_variance():
    P, _ = synth.random_instance(11, 1000, 3, 1, "uniform")
    r = oracle.lloyd(P, P[:1].astype(np.float64), max_iter=2, tol=-1, round_f32=False)
    P64 = P.astype(np.float64)
    np.testing.assert_allclose(r.centroids[0], P64.mean(0), rtol=1e-13)
    np.testing.assert_allclose(r.sse, len(P) * P64.var(0).sum(), rtol=1e-10)
    assert (r.labels == 0).all()


def test_k_equals_n_identity():
    P, _ = synth.random_instance(12, 50, 2, 1, "uniform")
    r = oracle.lloyd(P, P.astype(np.float64), max_iter=5, tol=0.0, round_f32=True)
    assert r.labels.tolist() == list(range(50))
    assert r.sse == 0.0 and r.iterations == 1 and r.drift_trace[0] == 0.0


@pytest.mark.parametrize("seed,d,k,kind", [(20, 2, 7, "blobs"), (21, 3, 25, "uniform"), (22, 2, 9, "grid"),
                                            (23, 3, 40, "offset")])
def test_invariants(seed, d, k, kind):
    P, C0 = synth.random_instance(seed, 1500, d, k, kind)
    C = C0.astype(np.float64)
    P64 = P.astype(np.float64)
    prev_sse = np.inf
    for t in range(6):
        a = oracle.assign(P, C)
        # brute force: full FP64 distance matrix, first index of the minimum
        D = ((P64[:, None, :] - C[None, :, :]) ** 2).sum(-1)
        np.testing.assert_array_equal(a.labels, D.argmin(1))
        np.testing.assert_allclose(a.best, D.min(1), rtol=1e-15, atol=0)
        u = oracle.update(P, a.labels, C, round_f32=True)
        assert u.counts.sum() == len(P)
        for j in range(k):
            m = a.labels == j
            want = P64[m].mean(0) if m.any() else C[j]
            np.testing.assert_allclose(u.centroids[j], want, rtol=2**-23, atol=0)
        s_t = a.best.sum()
        # SSE non-increasing; in mode A rounding the mean may add cnt*d*(ulp/2)^2
        slack = 1e-12 * prev_sse + len(P) * d * (np.spacing(np.abs(C).max().astype(np.float32)) / 2) ** 2
        assert s_t <= prev_sse + slack
        prev_sse = oracle.sse(P, a.labels, u.centroids)
        assert prev_sse <= s_t * (1 + 1e-12) + slack
        C = u.centroids


def test_permutation_equivariance_and_threads():
    P, C0 = synth.random_instance(30, 3000, 3, 20, "blobs")
    perm = np.random.default_rng(1).permutation(len(P))
    r1 = oracle.lloyd(P, C0.astype(np.float64), 8, -1.0, True, threads=1)
    r2 = oracle.lloyd(P[perm], C0.astype(np.float64), 8, -1.0, True, threads=oracle.max_threads())
    np.testing.assert_array_equal(r1.labels[perm], r2.labels)
    np.testing.assert_allclose(r1.centroids, r2.centroids, rtol=2**-23)
    r3 = oracle.lloyd(P, C0.astype(np.float64), 8, -1.0, True, threads=3)
    np.testing.assert_array_equal(r1.labels, r3.labels)
    np.testing.assert_array_equal(r1.centroids, r3.centroids)
    assert r1.sse == r3.sse


@pytest.mark.parametrize("order", ["big_first", "small_first", "big_last"])
def test_sse_sum_is_compensated(order):
    """SSE values (Eq. 1) are summed with Neumaier compensation,
    so the oracle's SSE equals the exactly rounded sum (math.fsum) where naive left-to-right
    summation loses every small term.  One point at distance 1e8 (D = 1e16, ulp 2) plus 1002
    points at distance 1: exact sum 1e16 + 1002 (representable); naive summation after the
    big term returns 1e16.  "small_first" puts one unit term before the big one, so the
    compensation's |x| > |s| branch takes the rounding error of 1 + 1e16; the three orders
    also catch a sign error in either branch.  Checked on oracle.sse (Eq. 1 of a given pair)
    and on the lloyd trace SSE_0 (same summation)."""
    import math
    big = np.array([[1e8, 0.0]], np.float32)
    unit = np.tile(np.array([[1.0, 0.0]], np.float32), (1002, 1))
    if order == "big_first":
        P = np.vstack([big, unit])
    elif order == "small_first":
        P = np.vstack([unit[:1], big, unit[1:]])
    else:
        P = np.vstack([unit, big])
    terms = [float(x) ** 2 for x in P[:, 0].astype(np.float64)]
    exact = math.fsum(terms)
    assert exact == 1e16 + 1002
    naive = 0.0
    for x in terms:
        naive += x
    if order != "big_last":
        assert naive != exact   # the fixture really separates the two
    lab = np.zeros(len(P), np.int32)
    C = np.zeros((1, 2))
    assert oracle.sse(P, lab, C) == exact
    r = oracle.lloyd(P, C, max_iter=1, tol=-1.0, round_f32=True)
    assert r.sse_trace[0] == exact
    a = oracle.assign(P, C)
    assert math.fsum(a.best.tolist()) == exact


def test_convergence_semantics():
    """tol < 0 runs exactly max_iter; tol = 0 stops at the fixpoint (R6)."""
    P, C0 = synth.random_instance(31, 400, 2, 5, "blobs")
    r = oracle.lloyd(P, C0.astype(np.float64), 15, -1.0, True)
    assert r.iterations == 15
    r0 = oracle.lloyd(P, C0.astype(np.float64), 200, 0.0, True)
    assert r0.iterations < 200
    last = r0.iterations - 1
    assert r0.drift_trace[last] == 0.0 or r0.changed_trace[last] == 0
    assert (r0.drift_trace[:last] > 0).all() and (r0.changed_trace[1:last] > 0).all()
    big = oracle.lloyd(P, C0.astype(np.float64), 50, 1e9, True)
    assert big.iterations == 1


# ---------------------------------------------- high-dimensional pins (NEXT-4, d = 128 / 256)
@pytest.mark.parametrize("dpad", [128, 256])
def test_high_d_zero_padding_is_exact(dpad):
    """Zero coordinates add exact 0 terms to every FP64 distance, sum and drift, so a d = 2 run
    padded to d = 128 / 256 must reproduce the (pinned) d = 2 run bit for bit: pins the
    d-generic loops of the oracle for the high-dimensional variant (Table tab:high_dimension,
    P:L636-671)."""
    P, C0 = synth.random_instance(40, 700, 2, 9, "blobs")
    Pp = np.zeros((len(P), dpad), np.float32)
    Pp[:, :2] = P
    Cp = np.zeros((9, dpad))
    Cp[:, :2] = C0
    a = oracle.lloyd(P, C0.astype(np.float64), 6, -1.0, True)
    b = oracle.lloyd(Pp, Cp, 6, -1.0, True)
    np.testing.assert_array_equal(a.labels, b.labels)
    np.testing.assert_array_equal(a.sse_trace, b.sse_trace)
    np.testing.assert_array_equal(a.changed_trace, b.changed_trace)
    np.testing.assert_array_equal(a.drift_trace, b.drift_trace)
    np.testing.assert_array_equal(a.centroids, b.centroids[:, :2])
    assert (b.centroids[:, 2:] == 0).all()


@pytest.mark.parametrize("seed", range(3))
def test_high_d_against_exact_rationals(seed):
    """d = 128 integer data: every FP64 distance is exact, so labels, best distances and
    counts equal the rational reference exactly, the means to FP64 rounding."""
    rng = np.random.default_rng(300 + seed)
    n, d, k = 30, 128, 3 + seed
    P = rng.integers(-3, 4, (n, d)).astype(np.float32)
    C0 = P[rng.choice(n, k, replace=False)].astype(np.float64)
    r = oracle.assign(P, C0)
    lab, best = pyref.assign(P.astype(int).tolist(), C0.astype(int).tolist())
    assert r.labels.tolist() == lab
    assert r.best.tolist() == [float(b) for b in best]
    u = oracle.update(P, r.labels, C0, round_f32=False)
    Cx, cnt = pyref.update(P.astype(int).tolist(), lab, C0.astype(int).tolist())
    assert u.counts.tolist() == cnt
    np.testing.assert_allclose(u.centroids, [[float(v) for v in c] for c in Cx], rtol=1e-15, atol=0)


@pytest.mark.parametrize("d,kind", [(128, "blobs"), (256, "uniform"), (128, "offset")])
def test_high_d_bruteforce_and_scipy(d, kind):
    """Labels = first argmin of the full FP64 distance matrix; mode B = scipy kmeans2."""
    P, C0 = synth.random_instance(41 + d, 600, d, 12, kind)
    C = C0.astype(np.float64)
    a = oracle.assign(P, C)
    P64 = P.astype(np.float64)
    D = ((P64[:, None, :] - C[None, :, :]) ** 2).sum(-1)
    np.testing.assert_array_equal(a.labels, D.argmin(1))
    np.testing.assert_allclose(a.best, D.min(1), rtol=1e-13, atol=0)
    cb, lab = _kmeans2(P, C0, 4)
    r = oracle.lloyd(P, C, max_iter=4, tol=-1, round_f32=False)
    np.testing.assert_array_equal(r.labels, lab)
    np.testing.assert_allclose(r.centroids, cb, rtol=1e-12, atol=1e-12)
