"""Shared comparison rules for GPU-vs-oracle parity.

North-star tolerances (BASELINE.json): labels identical except near-ties (best and
second-best squared distances within 1e-5 relative); centroids within 1e-4
relative; SSE within 1e-5 relative.  Reading R10 of "relative":
  centroid coordinate: |c_g - c_o| <= 1e-4 * max(|c_o|, 1e-3 * E), E = data extent.
Labels in LOCKSTEP (same float32 centroids on both sides) must be bit-identical:
libkm certifies every label against the FP64 distance.
"""
import numpy as np

import oracle

LABEL_REL = 1e-5
CENT_REL = 1e-4
SSE_REL = 1e-5


def extent(P):
    P = np.asarray(P, np.float64)
    return float((P.max(0) - P.min(0)).max()) if len(P) else 0.0


def assert_centroids_close(Cg, Co, P, rel=CENT_REL):
    Cg = np.asarray(Cg, np.float64)
    Co = np.asarray(Co, np.float64)
    floor = 1e-3 * max(extent(P), 1e-30)
    tol = rel * np.maximum(np.abs(Co), floor)
    bad = np.abs(Cg - Co) > tol
    assert not bad.any(), f"{bad.sum()} centroid coords out of tolerance; worst {np.abs(Cg - Co).max()}"
    return int((Cg != Co).sum())   # bit mismatches (reported, not gated)


def assert_sse_close(s_g, s_o, rel=SSE_REL):
    assert abs(s_g - s_o) <= rel * max(abs(s_o), 1e-300), f"SSE {s_g} vs {s_o}"


def assert_labels_near_tie_only(P, lab_g, C_prev, rel=LABEL_REL):
    """Free-run rule: a label may differ from the oracle's only where the oracle's
    best and second-best distances (against the centroids that assignment used)
    are within rel."""
    a = oracle.assign(P, np.asarray(C_prev, np.float64))
    diff = np.nonzero(np.asarray(lab_g) != a.labels)[0]
    if len(diff):
        gap = a.second[diff] - a.best[diff]
        ok = gap <= rel * np.maximum(a.best[diff], 1e-300)
        assert ok.all(), f"{(~ok).sum()} label mismatches that are not near-ties"
    return len(diff)
