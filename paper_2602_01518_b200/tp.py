"""Vocab-sharded (tensor-parallel LM-head) exact Top-k / Top-p — BASELINE config cfg5, SURVEY.md §8e.

Each rank holds a contiguous column shard ``[B, V_r]`` of the logits (columns
``[offset_r, offset_r + V_r)``, offsets increasing with rank).  The result on every rank is its shard
of the *unsharded* answer (oracle.py:70-89), bit-exact.

Exchange (one round, candidates instead of logits):

1. Local top-``min(k, V_r)`` on the shard with the B200 kernels (top-k only).  The global top-k set is
   a subset of the union of the local ones (a key above the k-th global key is above the local
   k-th on its own shard), and every quantity of the top-p stage — the row max, the normaliser over
   the survivors, their probabilities — depends only on that set (pipeline.py:226-239).
2. ``all_gather`` of the padded ``(value, global index)`` candidates: ``B x k`` per rank
   (cfg5: 128 x 1024 x 12 B = 1.5 MB per rank over NVLink).
3. Every rank re-runs the exact kernel on the gathered candidate rows, ordered by global index (so
   ties still break by global index), with the original k and p, and keeps its own columns.

Rows with ``k == V`` (top-p only) need the whole row's softmax normaliser; for those rows the
shards themselves are gathered (correct, communication-heavy; not a BASELINE case).

The local steps run through ``op`` (default: the CUDA ``topk_topp``); tests inject a CPU reference
op to exercise this protocol with ``gloo`` on machines without a GPU.
"""
from __future__ import annotations

from typing import Callable, List, Optional

import torch

PAD_VALUE = -3.4028234663852886e38  # -FLT_MAX: finite, below every real logit but -FLT_MAX itself


def _default_op():
    from .ops import topk_topp
    return lambda x, k, p: topk_topp(x, k, p)


class TorchComm:
    """all_gather over a torch.distributed process group (NCCL on B200s, gloo in tests)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def all_gather(self, t: torch.Tensor) -> List[torch.Tensor]:
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t.contiguous(), group=self.group)
        return out


def local_candidates(shard: torch.Tensor, k: torch.Tensor, offset: int, vocab: int,
                     op: Callable) -> tuple:
    """Top-min(k, V_r) of the shard as padded ``(values [B, kmax], global idx [B, kmax])``, with
    kmax = max(k) on every rank so the gathered pieces have one shape."""
    b, vr = shard.shape
    k_loc = torch.clamp(k, max=vr)
    ones = torch.ones(b, dtype=torch.float64, device=shard.device)
    masked = op(shard, k_loc, ones)
    keep = ~torch.isneginf(masked)
    kmax = max(1, min(int(k.max().item()) if b else 1, vocab))
    vals = torch.full((b, kmax), PAD_VALUE, dtype=torch.float32, device=shard.device)
    gidx = torch.full((b, kmax), vocab, dtype=torch.int64, device=shard.device)
    pos = torch.cumsum(keep.to(torch.int64), dim=1) - 1
    rr, cc = torch.nonzero(keep, as_tuple=True)
    vals[rr, pos[rr, cc]] = shard[rr, cc].to(torch.float32)
    gidx[rr, pos[rr, cc]] = cc + offset
    return vals, gidx


def resolve(vals: torch.Tensor, gidx: torch.Tensor, k: torch.Tensor, p: torch.Tensor,
            op: Callable, dtype: torch.dtype) -> tuple:
    """Exact answer on gathered candidate rows; returns (kept values, kept global idx, mask)."""
    order = torch.argsort(gidx, dim=1, stable=True)        # global index order; padding last
    g = torch.gather(gidx, 1, order)
    v = torch.gather(vals, 1, order).to(dtype)
    masked = op(v, torch.clamp(k, max=v.shape[1]), p)
    keep = ~torch.isneginf(masked)
    return v, g, keep


def topk_topp_tp(shard: torch.Tensor, k, p, *, vocab_offset: int, vocab_size: int,
                 comm=None, op: Optional[Callable] = None) -> torch.Tensor:
    """Exact truncation of a vocab shard; every rank returns its shard of the global answer."""
    comm = comm or TorchComm()
    op = op or _default_op()
    b, vr = shard.shape
    dev = shard.device
    k = torch.as_tensor(k, dtype=torch.int64, device=dev).expand(b).contiguous() if not \
        isinstance(k, torch.Tensor) or k.dim() == 0 else k.to(dev, torch.int64)
    p = torch.as_tensor(p, dtype=torch.float64, device=dev).expand(b).contiguous() if not \
        isinstance(p, torch.Tensor) or p.dim() == 0 else p.to(dev, torch.float64)
    out = torch.full_like(shard, float("-inf"))
    topp_only = k >= vocab_size
    part = ~topp_only
    if bool(part.any()):
        rows = torch.nonzero(part, as_tuple=True)[0]
        vals, gidx = local_candidates(shard[rows], k[rows], vocab_offset, vocab_size, op)
        all_v = comm.all_gather(vals)
        all_g = comm.all_gather(gidx)
        v, g, keep = resolve(torch.cat(all_v, 1), torch.cat(all_g, 1), k[rows], p[rows], op, shard.dtype)
        mine = keep & (g >= vocab_offset) & (g < vocab_offset + vr)
        rr, cc = torch.nonzero(mine, as_tuple=True)
        out[rows[rr], g[rr, cc] - vocab_offset] = v[rr, cc]
    if bool(topp_only.any()):
        rows = torch.nonzero(topp_only, as_tuple=True)[0]
        meta = comm.all_gather(torch.tensor([vocab_offset, vr], dtype=torch.int64, device=dev))
        wmax = max(int(m[1].item()) for m in meta)
        sub = torch.full((rows.numel(), wmax), PAD_VALUE, dtype=shard.dtype, device=dev)
        sub[:, :vr] = shard[rows]
        all_s = comm.all_gather(sub)
        order = sorted(range(len(all_s)), key=lambda i: int(meta[i][0].item()))
        full = torch.cat([all_s[i][:, :int(meta[i][1].item())] for i in order], 1)
        masked = op(full, torch.full((rows.numel(),), full.shape[1], dtype=torch.int64, device=dev), p[rows])
        out[rows] = masked[:, vocab_offset:vocab_offset + vr]
    return out


def simulate_tp(x: torch.Tensor, k, p, world: int, op: Optional[Callable] = None) -> torch.Tensor:
    """Run the TP protocol for `world` column shards of x inside one process (the candidate
    exchange becomes a concatenation).  Returns the full masked matrix."""
    op = op or _default_op()
    b, v = x.shape
    dev = x.device
    k = torch.as_tensor(k, dtype=torch.int64, device=dev).expand(b).contiguous() if not \
        isinstance(k, torch.Tensor) or k.dim() == 0 else k.to(dev, torch.int64)
    p = torch.as_tensor(p, dtype=torch.float64, device=dev).expand(b).contiguous() if not \
        isinstance(p, torch.Tensor) or p.dim() == 0 else p.to(dev, torch.float64)
    bounds = [v * r // world for r in range(world + 1)]
    shards = [x[:, bounds[r]:bounds[r + 1]].contiguous() for r in range(world)]
    topp_only = k >= v
    part = ~topp_only
    out = torch.full_like(x, float("-inf"))
    if bool(part.any()):
        rows = torch.nonzero(part, as_tuple=True)[0]
        cands = [local_candidates(shards[r][rows], k[rows], bounds[r], v, op) for r in range(world)]
        vals = torch.cat([c[0] for c in cands], 1)
        gidx = torch.cat([c[1] for c in cands], 1)
        vv, g, keep = resolve(vals, gidx, k[rows], p[rows], op, x.dtype)
        rr, cc = torch.nonzero(keep, as_tuple=True)
        out[rows[rr], g[rr, cc]] = vv[rr, cc]
    if bool(topp_only.any()):
        rows = torch.nonzero(topp_only, as_tuple=True)[0]
        out[rows] = op(x[rows], k[rows], p[rows])
    return out
