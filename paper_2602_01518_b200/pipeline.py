"""Per-row entry points — the reference's pipeline.py surface (pkg/src/sigmatop/pipeline.py:140-239).

Each call is a batch of one row through the same B200 kernels as run_batch.  Argument checks and
their ValueError texts follow the reference (pipeline.py:148-149, 168-169, 208-211).  Rows may be
numpy arrays (result is numpy, in the row's dtype) or 1-D CUDA tensors (result stays on the device).
"""
from __future__ import annotations

import numpy as np
import torch

from . import ops
from .core import DEFAULT_TOL, RowMetrics, Tolerances, TruncationOutput, _is_tensor
from .engine import metrics_to_rows

__all__ = ["truncate_topk", "truncate_topp", "truncate_topk_topp"]


def _run_row(row, k: int, p: float, *, search, use_sigma_trunc, force_fallback, dup_handling,
             sample_size, inplace) -> TruncationOutput:
    is_t = _is_tensor(row)
    if is_t:
        x = row if row.is_cuda else row.to("cuda")
    else:
        arr = np.asarray(row)
        x = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float32)).to("cuda")
    if x.dim() != 1:
        raise ValueError("row must be 1-D")
    if x.dtype not in (torch.float32, torch.bfloat16):
        x = x.to(torch.float32)
    x2 = x.unsqueeze(0)
    flags = ops.TruncFlags(search=search, use_sigma_trunc=use_sigma_trunc,
                           force_fallback=force_fallback, dup_handling=dup_handling)
    met = ops.metrics_buffer(1, x.device)
    kept = torch.zeros(1, dtype=torch.int32, device=x.device)
    dev_inplace = inplace and is_t and row.is_cuda and x.data_ptr() == row.data_ptr()
    out = ops.topk_topp(x2, int(k), float(p), inplace=dev_inplace, flags=flags,
                        sample_size=sample_size, kept_count=kept, metrics=met, check=True)
    metrics = metrics_to_rows(met)[0]
    kept_count = int(kept.item())
    if is_t:
        masked = out[0]
        if inplace and not dev_inplace:
            row.copy_(masked)
            masked = row
    else:
        res = out[0].cpu().numpy()
        if inplace:
            arr[...] = res.astype(arr.dtype, copy=False)
            masked = arr
        else:
            masked = res.astype(arr.dtype, copy=False) if arr.dtype != np.float32 else res
    return TruncationOutput(masked_row=masked, kept_count=kept_count, metrics=metrics)


def _check_k(k: int, v: int):
    if not 1 <= k <= v:
        raise ValueError(f"k must be in [1, V], got k={k}, V={v}")


def _check_p(p: float):
    if not 0.0 < p <= 1.0:
        raise ValueError(f"p must be in (0, 1], got {p}")


def truncate_topk(row, k: int, tol: Tolerances = DEFAULT_TOL, *, search: str = "quaternary",
                  use_sigma_trunc: bool = True, force_fallback: bool = False,
                  dup_handling: bool = True, sample_size: int = ops.DEFAULT_SAMPLE_SIZE,
                  inplace: bool = False) -> TruncationOutput:
    """Keep exactly the k largest entries, ties to earlier indices (pipeline.py:140-158)."""
    v = int(row.shape[0])
    _check_k(k, v)
    return _run_row(row, k, 1.0, search=search, use_sigma_trunc=use_sigma_trunc,
                    force_fallback=force_fallback, dup_handling=dup_handling,
                    sample_size=sample_size, inplace=inplace)


def truncate_topp(row, p: float, tol: Tolerances = DEFAULT_TOL, *, search: str = "quaternary",
                  use_sigma_trunc: bool = True, force_fallback: bool = False,
                  dup_handling: bool = True, sample_size: int = ops.DEFAULT_SAMPLE_SIZE,
                  inplace: bool = False) -> TruncationOutput:
    """Minimal set of highest-probability entries with mass >= p (pipeline.py:161-196)."""
    _check_p(p)
    v = int(row.shape[0])
    return _run_row(row, v, p, search=search, use_sigma_trunc=use_sigma_trunc,
                    force_fallback=force_fallback, dup_handling=dup_handling,
                    sample_size=sample_size, inplace=inplace)


def truncate_topk_topp(row, k: int, p: float, tol: Tolerances = DEFAULT_TOL, *,
                       search: str = "quaternary", use_sigma_trunc: bool = True,
                       force_fallback: bool = False, dup_handling: bool = True,
                       sample_size: int = ops.DEFAULT_SAMPLE_SIZE,
                       inplace: bool = False) -> TruncationOutput:
    """Top-k first, then top-p over the softmax renormalised on the survivors (pipeline.py:199-239)."""
    v = int(row.shape[0])
    _check_k(k, v)
    _check_p(p)
    return _run_row(row, k, p, search=search, use_sigma_trunc=use_sigma_trunc,
                    force_fallback=force_fallback, dup_handling=dup_handling,
                    sample_size=sample_size, inplace=inplace)
