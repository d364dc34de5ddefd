"""LM-head producer fusion: the bf16 LM-head GEMM whose epilogue runs the
truncation's streaming pass, so that on a sigma hit the fp32 logits are written once and never read
back (csrc/qrita_lmhead.cu).  The reference has no code for this producer; the consumer semantics are
truncate_topk_topp (pkg/src/sigmatop/pipeline.py:199-239) / oracle_topk_topp (oracle.py:70-89), and
the kept sets equal topk_topp_indices on the same logits, bit for bit."""
from __future__ import annotations

import ctypes
from typing import Optional, Tuple, Union

import torch

from . import _native as N
from .ops import TruncFlags, _per_row, check_status, workspace_for

__all__ = ["lm_head_logits", "lm_head_topk_topp"]


def _check(hidden: torch.Tensor, weight: torch.Tensor) -> Tuple[int, int, int]:
    for name, t in (("hidden", hidden), ("weight", weight)):
        if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.bfloat16 or t.dim() != 2:
            raise TypeError(f"{name} must be a 2-D bfloat16 CUDA tensor")
        if t.stride(1) != 1 or (t.stride(0) * 2) % 16 or t.data_ptr() % 16:
            raise ValueError(f"{name} needs unit column stride and 16-byte aligned rows")
    b, d = hidden.shape
    v, d2 = weight.shape
    if d != d2:
        raise ValueError(f"hidden size mismatch: hidden has {d}, weight has {d2}")
    if d % 64 or b < 1 or v < 1:
        raise ValueError("need B >= 1, V >= 1 and a hidden size that is a multiple of 64")
    if hidden.device != weight.device:
        raise ValueError("hidden and weight must be on the same device")
    return b, v, d


def lm_head_logits(hidden: torch.Tensor, weight: torch.Tensor, *, out: Optional[torch.Tensor] = None,
                   stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """fp32 logits = hidden @ weight.T on the tensor cores (tcgen05, bf16 inputs, fp32 accumulation)."""
    b, v, d = _check(hidden, weight)
    dev = hidden.device
    st = stream or torch.cuda.current_stream(dev)
    with torch.cuda.device(dev), torch.cuda.stream(st):
        if out is None:
            out = torch.empty((b, v), dtype=torch.float32, device=dev)
        elif out.dtype != torch.float32 or out.shape != (b, v) or out.stride(1) != 1:
            raise ValueError("out must be float32 [B, V] with unit column stride")
        rc = N.load().qrita_lmhead_logits(
            ctypes.c_void_p(hidden.data_ptr()), hidden.stride(0), ctypes.c_void_p(weight.data_ptr()),
            weight.stride(0), b, v, d, ctypes.c_void_p(out.data_ptr()), out.stride(0),
            ctypes.c_void_p(st.cuda_stream))
    if rc != N.OK:
        raise RuntimeError(f"qrita_lmhead_logits failed: {N.strerror(rc)}")
    return out


def lm_head_topk_topp(hidden: torch.Tensor, weight: torch.Tensor, k: Union[int, torch.Tensor],
                      p: Union[float, torch.Tensor], *, flags: Optional[TruncFlags] = None,
                      metrics: Optional[torch.Tensor] = None, check: bool = False, k_cap: Optional[int] = None,
                      stream: Optional[torch.cuda.Stream] = None
                      ) -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """LM head + exact Top-k / Top-p in one pipeline.  Returns (logits fp32 [B, V], kept_idx int32
    [B, V] — or [B, k_cap] with k_cap —, kept_count int32 [B]); row r keeps
    logits[r, kept_idx[r, :kept_count[r]]] (unordered), the set topk_topp_indices(logits, k, p)
    returns.  k_cap: compact kept lists for batches whose rows are all top-k rows with k <= k_cap < V
    (checked, one synchronisation).  Stream-ordered; check=True synchronises and raises the reference's
    ValueError for invalid rows."""
    b, v, d = _check(hidden, weight)
    dev = hidden.device
    fl = (flags or TruncFlags()).bits()
    st = stream or torch.cuda.current_stream(dev)
    lib = N.load()
    need = lib.qrita_lmhead_workspace_bytes(b, v)
    ws = workspace_for(dev, st)
    with torch.cuda.device(dev), torch.cuda.stream(st):
        kt = _per_row(k, b, torch.int64, dev, "k")
        pt = _per_row(p, b, torch.float64, dev, "p")
        logits = torch.empty((b, v), dtype=torch.float32, device=dev)
        ld_idx = v
        if k_cap is not None:
            kmax = int(kt.max().item())
            if not (1 <= int(kt.min().item()) and kmax <= int(k_cap) < v):
                raise ValueError(f"k_cap={k_cap} needs every row to be a top-k row with k <= k_cap < V "
                                 f"(max k {kmax}, V {v})")
            ld_idx = int(k_cap)
        kept_idx = torch.empty((b, ld_idx), dtype=torch.int32, device=dev)
        kept_count = torch.empty((b,), dtype=torch.int32, device=dev)
        ws_ptr, ws_bytes = ws.get(need, st)
        rc = lib.qrita_lmhead_topk_topp(
            ctypes.c_void_p(hidden.data_ptr()), hidden.stride(0), ctypes.c_void_p(weight.data_ptr()),
            weight.stride(0), b, v, d, ctypes.c_void_p(kt.data_ptr()), ctypes.c_void_p(pt.data_ptr()),
            ctypes.c_void_p(logits.data_ptr()), v, ctypes.c_void_p(kept_idx.data_ptr()), ld_idx,
            ctypes.c_void_p(kept_count.data_ptr()), ctypes.c_void_p(metrics.data_ptr() if metrics is not None else 0),
            ctypes.c_void_p(ws_ptr), ws_bytes, fl, ctypes.c_void_p(st.cuda_stream))
        if rc != N.OK:
            ws.reset()
            raise RuntimeError(f"qrita_lmhead_topk_topp failed: {N.strerror(rc)}")
        if check:
            check_status(ws_ptr, b, logits, kt, pt, st)
    return logits, kept_idx, kept_count
