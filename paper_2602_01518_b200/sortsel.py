"""Sort-based Top-k / Top-p on the GPU with plain torch ops — the comparison baselines.

* `exact_sort_topk_topp` — the reference's definition computed the slow way (engine.sort_select,
  engine.py:183-205, over oracle.py:70-89): stable descending sort, top-k prefix, fp64 softmax over
  the survivors, exact fixed-point prefix masses, first crossing.  An implementation independent of
  the pivot-search kernels, used as verify_batch's default reference.
* `torch_sort_topk_topp` — the common serving-stack recipe (sort, mask k, fp32 softmax, cumsum, mask
  p, scatter back) that BASELINE.md's "torch.sort-based GPU baseline" refers to.  Not exact: fp32
  cumsum flips 8-17% of rows; it is a throughput yardstick only.
"""
from __future__ import annotations

import math
import struct
from fractions import Fraction

import torch

_UNIT = 128          # fixed point unit 2^-128
_LIMBS = 5           # 32-bit limbs -> 160 bits, integer part < 2^32
_MASK = (1 << 32) - 1


def _to_limbs(x: torch.Tensor) -> torch.Tensor:
    """fp64 >= 0 -> [..., 5] int64 limbs of floor(x * 2^128) (truncated below 2^-128)."""
    mant, ex = torch.frexp(x)                     # x = mant * 2^ex, mant in [0.5, 1)
    M = torch.ldexp(mant, torch.full_like(ex, 53)).to(torch.int64)   # exact 53-bit integer
    s = ex.to(torch.int64) - 53 + _UNIT           # x * 2^128 = M * 2^s
    limbs = []
    for i in range(_LIMBS):
        t = s - 32 * i
        pos = t >= 0
        tp = t.clamp(0, 31)
        left = torch.where(t < 32, (M & ((1 << (32 - tp)) - 1)) << tp, torch.zeros_like(M))
        tn = (-t).clamp(0, 63)
        right = (M >> tn) & _MASK
        limbs.append(torch.where(pos, left, right))
    out = torch.stack(limbs, dim=-1)
    return torch.where((x > 0).unsqueeze(-1), out, torch.zeros_like(out))


def _normalize(l: torch.Tensor) -> torch.Tensor:
    """Propagate carries of lazily summed 32-bit limbs (last dim)."""
    parts = []
    carry = torch.zeros_like(l[..., 0])
    for i in range(_LIMBS):
        v = l[..., i] + carry
        parts.append(v & _MASK)
        carry = v >> 32
    return torch.stack(parts, dim=-1)


def _limbs_of_int(v: int, device) -> torch.Tensor:
    return torch.tensor([(v >> (32 * i)) & _MASK for i in range(_LIMBS)], dtype=torch.int64,
                        device=device)


def _ge(a: torch.Tensor, t: torch.Tensor) -> torch.Tensor:
    """Lexicographic a >= t over normalized limbs (most significant last)."""
    res = torch.ones(a.shape[:-1], dtype=torch.bool, device=a.device)
    for i in range(_LIMBS):  # from least to most significant: later limbs override
        gt = a[..., i] > t[..., i]
        lt = a[..., i] < t[..., i]
        res = torch.where(gt, torch.ones_like(res), torch.where(lt, torch.zeros_like(res), res))
    return res


def _round_threshold(p: float) -> int:
    """Smallest integer multiple S of 2^-128 (as an int) with fsum-rounding(S) >= p."""
    if p < 2.0 ** -70:
        return 1
    q = math.nextafter(p, 0.0)
    P = Fraction(p) * (1 << _UNIT)
    Q = Fraction(q) * (1 << _UNIT)
    mid = (P + Q) / 2
    assert mid.denominator == 1
    mid = int(mid)
    even = (struct.unpack("<Q", struct.pack("<d", p))[0] & 1) == 0  # ties-to-even picks p
    return mid if even else mid + 1


@torch.no_grad()
def exact_sort_topk_topp(x: torch.Tensor, k: torch.Tensor, p: torch.Tensor,
                         rows_per_step: int = 64, dup_handling: bool = True) -> torch.Tensor:
    """Exact reference semantics via a stable sort; returns masked logits in x's dtype.
    dup_handling=False: the reference pipeline's whole-cluster rule (pipeline.py:47-57; Table 3
    runs C / E): each stage keeps every copy of its boundary value."""
    b, v = x.shape
    out = torch.full_like(x, float("-inf"))
    kk = k.tolist()
    pp = p.tolist()
    for r0 in range(0, b, rows_per_step):
        r1 = min(b, r0 + rows_per_step)
        z = x[r0:r1].to(torch.float64) + 0.0      # -0.0 -> +0.0 so ties are exact
        zs, order = torch.sort(z, dim=1, descending=True, stable=True)
        m = zs[:, :1]
        for i in range(r1 - r0):
            r = r0 + i
            ki, pi = int(kk[r]), float(pp[r])
            if ki == v and pi == 1.0:
                out[r] = x[r]
                continue
            if not dup_handling and ki < v:   # the whole k-th cluster survives
                ki = int((zs[i] >= zs[i, ki - 1]).sum())
            if pi == 1.0:
                idx = order[i, :ki]
                out[r, idx] = x[r, idx]
                continue
            e = torch.exp(zs[i, :ki] - m[i])
            D_int = _normalize(_to_limbs(e).sum(dim=0))
            D = Fraction(sum(int(D_int[j]) << (32 * j) for j in range(_LIMBS)), 1 << _UNIT)
            D = float(D)
            probs = e / D
            pref = _normalize(torch.cumsum(_to_limbs(probs), dim=0))
            t_p = _limbs_of_int(_round_threshold(pi), x.device)
            t_sp = _limbs_of_int(_round_threshold(math.nextafter(pi, 2.0)), x.device)
            if not bool(_ge(pref[-1], t_sp)):
                L = ki
            else:
                L = int(torch.nonzero(_ge(pref, t_p))[0, 0]) + 1
                if not dup_handling:          # and the whole crossing cluster
                    L = int((zs[i, :ki] >= zs[i, L - 1]).sum())
            idx = order[i, :L]
            out[r, idx] = x[r, idx]
    return out


@torch.no_grad()
def torch_sort_topk_topp(x: torch.Tensor, k: torch.Tensor, p: torch.Tensor) -> torch.Tensor:
    """Serving-stack recipe: sort ascending, mask below the k-th, softmax, cumsum, mask p, scatter."""
    logits_sort, idx = x.sort(dim=-1, descending=False)
    v = x.shape[1]
    top_k_mask = logits_sort.gather(1, (v - k.to(torch.long)).unsqueeze(1))
    logits_sort = logits_sort.masked_fill(logits_sort < top_k_mask, float("-inf"))
    probs_sort = logits_sort.softmax(dim=-1)
    probs_sum = torch.cumsum(probs_sort, dim=-1, out=probs_sort)
    top_p_mask = probs_sum <= 1 - p.to(probs_sum.dtype).unsqueeze(1)
    top_p_mask[:, -1] = False
    logits_sort = logits_sort.masked_fill(top_p_mask, float("-inf"))
    return logits_sort.scatter(dim=-1, index=idx, src=logits_sort)
