"""The reference's pivot_search and oracle surfaces (pkg/src/sigmatop/pivot_search.py, oracle.py) for
drop-in callers, computed exactly on the GPU.

The fused kernel never runs the reference's floating-point pivot iterations: it searches integer
order keys with exact fixed-point masses.  These standalone functions keep the
reference's names, dataclasses, argument checks and early exits, and return the EXACT boundary the
reference's search converges to (its terminal condition: N >= k and N - n_dup < k for top-k,
S >= p and S - S_dup < p resolved with fsum for top-p, pivot_search.py:113-116, 143-196), from one
stable sort on the GPU.  Ties are exact equality (the oracle's rule) instead of eq_eps; `iters`
reports 1 (one sort) — trajectories are not reproduced.

``oracle_topk`` / ``oracle_topp`` / ``oracle_topk_topp`` (oracle.py:28-89) are the sort-based
definition on the GPU (sortsel.exact_sort_topk_topp).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from fractions import Fraction

import numpy as np
import torch

from .core import DEFAULT_TOL, Tolerances, TruncationOutput, _is_tensor
from .sortsel import _LIMBS, _UNIT, _ge, _limbs_of_int, _normalize, _round_threshold, _to_limbs


@dataclass(frozen=True)
class PivotResult:
    """Top-k search outcome (pivot_search.py:18-32)."""

    tau: float
    n_above: int
    z_dup: float
    n_dup: int
    iters: int = 0
    ties_only: bool = False


@dataclass(frozen=True)
class NucleusPivotResult:
    """Top-p search outcome in probability space (pivot_search.py:35-49)."""

    pi: float
    s_above: float
    p_mn: float
    n_dup: int
    n_keep: int
    iters: int = 0


def _values(values) -> torch.Tensor:
    t = values if _is_tensor(values) else torch.as_tensor(np.asarray(values, dtype=np.float64))
    t = t.to(device="cuda", dtype=torch.float64).reshape(-1)
    if t.shape[0] == 0:
        raise ValueError("pivot search requires a non-empty value set")
    return t + 0.0   # -0.0 -> +0.0


def _search_topk(values, k: int, lo, hi) -> PivotResult:
    v = _values(values)
    l = float(v.min()) if lo is None else float(lo)
    r = float(v.max()) if hi is None else float(hi)
    n_all = v.shape[0]
    if not 1 <= k <= n_all:
        raise ValueError("k must be in [1, |values|]")
    if l == r:
        return PivotResult(tau=l, n_above=0, z_dup=l, n_dup=n_all, iters=0, ties_only=True)
    if k > int((v > l).sum()):
        # pivot_search.py:102-106: tau = -inf, keep everything, trim the minimum's copies
        z_mn = float(v.min())
        return PivotResult(tau=-math.inf, n_above=n_all, z_dup=z_mn, n_dup=int((v == z_mn).sum()), iters=0)
    s, _ = torch.sort(v, descending=True, stable=True)
    z_b = float(s[k - 1])
    below = s[s < z_b]
    tau = max(l, float(below[0])) if below.numel() else l
    n_above = int((v > tau).sum())
    return PivotResult(tau=tau, n_above=n_above, z_dup=z_b, n_dup=int((v == z_b).sum()), iters=1)


def quaternary_topk(values, k: int, tol: Tolerances = DEFAULT_TOL, lo: float = None, hi: float = None) -> PivotResult:
    return _search_topk(values, k, lo, hi)


def binary_topk(values, k: int, tol: Tolerances = DEFAULT_TOL, lo: float = None, hi: float = None) -> PivotResult:
    return _search_topk(values, k, lo, hi)


def _fx_to_float(limbs: torch.Tensor) -> float:
    n = sum(int(limbs[j]) << (32 * j) for j in range(_LIMBS))
    return float(Fraction(n, 1 << _UNIT))


def _search_topp(probs, p: float, lo, hi) -> NucleusPivotResult:
    v = _values(probs)
    if not 0.0 < p < 1.0:
        raise ValueError("p must be in (0, 1)")
    s, _ = torch.sort(v, descending=True, stable=True)
    pref = _normalize(torch.cumsum(_to_limbs(s), dim=0))           # exact prefix masses
    total = _fx_to_float(pref[-1])
    t_p = _limbs_of_int(_round_threshold(p), v.device)
    if not bool(_ge(pref[-1], t_p)):
        # pivot_search.py:182-185: even the whole set falls short of p -> keep all
        return NucleusPivotResult(pi=0.0, s_above=total, p_mn=0.0, n_dup=0, n_keep=0, iters=0)
    L = int(torch.nonzero(_ge(pref, t_p))[0, 0]) + 1
    p_mn = float(s[L - 1])
    n_dup = int((v == p_mn).sum())
    n_head = int((v > p_mn).sum())
    s_all = _fx_to_float(pref[n_head + n_dup - 1])
    return NucleusPivotResult(pi=p_mn * (1.0 - 2.0 * DEFAULT_TOL.eq_eps), s_above=s_all, p_mn=p_mn, n_dup=n_dup,
                              n_keep=L - n_head, iters=1)


def quaternary_topp(probs, p: float, tol: Tolerances = DEFAULT_TOL, lo: float = None,
                    hi: float = None) -> NucleusPivotResult:
    return _search_topp(probs, p, lo, hi)


def binary_topp(probs, p: float, tol: Tolerances = DEFAULT_TOL, lo: float = None,
                hi: float = None) -> NucleusPivotResult:
    return _search_topp(probs, p, lo, hi)


def _oracle_row(row, k: int, p: float) -> TruncationOutput:
    from .sortsel import exact_sort_topk_topp
    is_t = _is_tensor(row)
    x = row if is_t else torch.from_numpy(np.ascontiguousarray(np.asarray(row)))
    x = x.to("cuda").reshape(1, -1)
    if x.dtype not in (torch.float32, torch.bfloat16):
        x = x.to(torch.float32)
    v = x.shape[1]
    if not 1 <= k <= v:
        raise ValueError(f"k must be in [1, V], got k={k}, V={v}")
    if not 0.0 < p <= 1.0:
        raise ValueError(f"p must be in (0, 1], got {p}")
    out = exact_sort_topk_topp(x, torch.tensor([k], device=x.device), torch.tensor([p], dtype=torch.float64,
                                                                                    device=x.device))[0]
    kept = int((~torch.isneginf(out)).sum())
    if not is_t:
        arr = np.asarray(row)
        out = out.cpu().numpy().astype(arr.dtype, copy=False)
    return TruncationOutput(masked_row=out, kept_count=kept)


def oracle_topk(row, k: int) -> TruncationOutput:
    """Stable descending sort, keep the first k (oracle.py:28-34), on the GPU."""
    return _oracle_row(row, int(k), 1.0)


def oracle_topp(row, p: float) -> TruncationOutput:
    """Shortest descending prefix whose fsum mass reaches p (oracle.py:57-67), on the GPU."""
    v = (row.shape[-1] if _is_tensor(row) else np.asarray(row).shape[-1])
    return _oracle_row(row, int(v), float(p))


def oracle_topk_topp(row, k: int, p: float) -> TruncationOutput:
    """Top-k, then top-p renormalised over the survivors (oracle.py:70-89), on the GPU."""
    return _oracle_row(row, int(k), float(p))


__all__ = ["PivotResult", "NucleusPivotResult", "quaternary_topk", "binary_topk", "quaternary_topp",
           "binary_topp", "oracle_topk", "oracle_topp", "oracle_topk_topp"]
