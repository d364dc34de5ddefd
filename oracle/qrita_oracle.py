"""CPU oracle for exact Top-k / Top-p truncation — TEST INFRASTRUCTURE ONLY.

Nothing in the product package (`paper_2602_01518_b200/`) imports this module.  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s CPU-baseline leg (`cpu_baseline` / `--impl reference`)
use it, and only as the checker or the timed CPU reference — never as the thing shipped.

It restates the ground-truth semantics of the reference (arxiv/paper_2602_01518, package
`sigmatop`) with numpy:

* stable descending order, ties to the lower index, -0.0 == +0.0 ........ oracle.py:16-18
* top-k = the first k of that order ...................................... oracle.py:28-34
* fp64 softmax: m = row max, e = exp(z - m), D = pairwise sum ............ core.py:93-103
* nucleus = shortest prefix whose exactly-rounded (fsum) mass reaches p;
  keep everything when p >= fsum(all) ................................... oracle.py:37-54
* top-p only (k == V): softmax over the whole row ........................ oracle.py:57-67
* combined: top-k survivors, softmax renormalised over the survivors with
  the full-row max and the denominator summed in index order ............ oracle.py:70-89
* k == V and p == 1: copy; k == V: top-p only; p == 1: top-k only ........ oracle.py:62-64, 78-81

Pinning: `tests/test_oracle_golden.py` checks this restatement against golden vectors produced by
the reference itself (`tests/golden/make_golden.py`, run where `/root/reference` is mounted):
the reference's unit-test known answers, an exhaustive small-row corpus, an acceptance-style corpus,
and every BASELINE config.  Probability bits depend on the host's numpy `exp`, so
parity is pinned on kept-index sets, not on probability ulps.
"""
from __future__ import annotations

import math

import numpy as np

__all__ = [
    "stable_desc_order", "nucleus_length", "oracle_keep_row", "oracle_batch", "boundary_of_mask",
    "mask_from_boundary", "crossing_margin", "oracle_keep_row_nodup",
]


def stable_desc_order(row: np.ndarray) -> np.ndarray:
    """Indices by (value desc, index asc); float64 negation makes -0.0 and +0.0 equal (oracle.py:16-18)."""
    return np.argsort(-np.asarray(row, dtype=np.float64), kind="stable")


def nucleus_length(sorted_probs: np.ndarray, p: float) -> int:
    """Length of the shortest prefix with fsum >= p; all of it when p >= fsum(all) (oracle.py:37-54)."""
    vals = sorted_probs.tolist()
    if p >= math.fsum(vals):
        return len(vals)
    lo, hi = 1, len(vals)
    while lo < hi:
        mid = (lo + hi) // 2
        if math.fsum(vals[:mid]) >= p:
            hi = mid
        else:
            lo = mid + 1
    return lo


def oracle_keep_row(row: np.ndarray, k: int, p: float) -> np.ndarray:
    """Boolean kept mask of one row under the reference semantics (oracle.py:70-89)."""
    row = np.asarray(row)
    v = row.shape[0]
    if not 1 <= k <= v:
        raise ValueError(f"k must be in [1, V], got k={k}, V={v}")
    if not 0.0 < p <= 1.0:
        raise ValueError(f"p must be in (0, 1], got {p}")
    keep = np.zeros(v, dtype=bool)
    if k == v and p == 1.0:
        keep[:] = True
        return keep
    order = stable_desc_order(row)
    if p == 1.0:
        keep[order[:k]] = True
        return keep
    z = row.astype(np.float64)
    m = float(z.max())
    if k == v:
        # full-row softmax (core.py:93-103): numpy exp, pairwise sum in index order
        e = np.exp(z - m)
        denom = float(e.sum())
        survivors = order
        probs_desc = (e / denom)[order]
    else:
        survivors = order[:k]
        denom = float(np.exp(z[np.sort(survivors)] - m).sum())
        probs_desc = np.exp(z[survivors] - m) / denom
    length = nucleus_length(probs_desc, float(p))
    keep[survivors[:length]] = True
    return keep


def oracle_keep_row_nodup(row: np.ndarray, k: int, p: float) -> np.ndarray:
    """Kept mask of the reference PIPELINE with duplication_handling_enabled=False (Table 3 runs C /
    E): each stage keeps its whole boundary cluster (pipeline.py:47-57 skips the occurrence trim):
    the top-k stage keeps every z >= z_k (the k-th value of the stable order); the top-p stage
    renormalises over those survivors with the full-row max (pipeline.py:226-239) and keeps every
    survivor >= the value at which the exactly rounded prefix mass crosses p (pivot_search.py:159-196
    keeps all when even the whole set falls short)."""
    row = np.asarray(row)
    v = row.shape[0]
    z = row.astype(np.float64)
    keep = np.ones(v, dtype=bool)
    order = stable_desc_order(row)
    if k < v:
        keep = z >= z[order[k - 1]]
    if p == 1.0:
        return keep
    m = float(z.max())
    surv = np.nonzero(keep)[0]                      # index order
    e = np.exp(z[surv] - m)
    denom = float(e.sum())
    probs = e / denom
    o = np.argsort(-z[surv], kind="stable")
    length = nucleus_length(probs[o], float(p))
    zb = z[surv][o[length - 1]]
    return keep & (z >= zb)


def oracle_batch(x: np.ndarray, k, p):
    """Masked [B, V] output (input dtype, -inf outside the kept set) and kept counts."""
    x = np.asarray(x)
    b = x.shape[0]
    k = np.broadcast_to(np.asarray(k, dtype=np.int64), (b,))
    p = np.broadcast_to(np.asarray(p, dtype=np.float64), (b,))
    out = np.full_like(x, -np.inf)
    counts = np.zeros(b, dtype=np.int64)
    for i in range(b):
        keep = oracle_keep_row(x[i], int(k[i]), float(p[i]))
        out[i, keep] = x[i, keep]
        counts[i] = int(keep.sum())
    return out, counts


def boundary_of_mask(row: np.ndarray, keep: np.ndarray):
    """Compact exact description of a kept set: (boundary value bits, last kept index of the boundary
    cluster, kept count).  kept(i) <=> z_i > z_b or (z_i == z_b and i <= cut)."""
    row32 = np.asarray(row, dtype=np.float32)
    kept_vals = row32[keep].astype(np.float64)
    zb = np.float32(kept_vals.min())
    cluster = np.nonzero(keep & (row32.astype(np.float64) == float(zb)))[0]
    cut = int(cluster.max())
    return int(np.float32(zb).view(np.uint32)), cut, int(keep.sum())


def mask_from_boundary(row: np.ndarray, zb_bits: int, cut: int) -> np.ndarray:
    row64 = np.asarray(row, dtype=np.float32).astype(np.float64)
    zb = float(np.uint32(zb_bits).view(np.float32))
    idx = np.arange(row64.shape[0])
    return (row64 > zb) | ((row64 == zb) & (idx <= cut))


def crossing_margin(row: np.ndarray, k: int, p: float) -> float:
    """Relative distance between p and the two prefix sums that straddle the nucleus crossing
    (SURVEY.md §8c audit).  Rows with a margin below ~1e-13 are 'ulp-sensitive': their kept set
    may legitimately depend on the last bit of exp()."""
    row = np.asarray(row)
    v = row.shape[0]
    if p == 1.0:
        return math.inf
    order = stable_desc_order(row)
    z = row.astype(np.float64)
    m = float(z.max())
    if k == v:
        e = np.exp(z - m)
        probs_desc = (e / float(e.sum()))[order]
    else:
        s = order[:k]
        probs_desc = np.exp(z[s] - m) / float(np.exp(z[np.sort(s)] - m).sum())
    vals = probs_desc.tolist()
    if p >= math.fsum(vals):
        return abs(math.fsum(vals) - p) / p
    length = nucleus_length(probs_desc, p)
    hi = math.fsum(vals[:length])
    lo = math.fsum(vals[:length - 1]) if length > 1 else 0.0
    return min(abs(hi - p), abs(p - lo)) / p
