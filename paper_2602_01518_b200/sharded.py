"""Row-sharded multi-GPU truncation (BASELINE config cfg4).

Rows are independent and their output slots are disjoint (pkg/src/sigmatop/engine.py:82-101; SPEC
"results are invariant to thread count"), so a batch shards by contiguous row blocks, one block per
device, with no collective on the data path.  Two ways to run it:

* one process per GPU (torchrun / bench.py --gpus N): every rank takes ``rank_rows(B, rank, world)``
  of the batch and truncates it with the single-device operator; ``aggregate_max`` turns the
  per-rank times into the job time (max over ranks);
* one process driving several devices: ``topk_topp_sharded(logits, k, p, devices=[...])`` splits the
  rows into contiguous blocks and runs each block on its own device (and stream), one host thread
  per block.  Host tensors go through the native host-buffer pipeline of each device
  (``qrita_topk_topp_host``: every GPU pulls its rows over its own PCIe link); CUDA tensors are
  copied block-wise to their devices and the results copied back.

The same device may appear more than once in ``devices`` (each block then gets its own stream and
workspace) — that is how the sharded path is tested on a single GPU.
"""
from __future__ import annotations

import contextlib
import threading
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import ops


def row_blocks(b: int, n: int) -> List[Tuple[int, int]]:
    """Contiguous, balanced row blocks ``[lo, hi)`` of a B-row batch over n shards (sizes differ by at
    most one; block i starts at floor(B*i/n))."""
    if b < 0 or n < 1:
        raise ValueError("need B >= 0 and n >= 1")
    return [(b * i // n, b * (i + 1) // n) for i in range(n)]


def rank_rows(b: int, rank: int, world: int) -> Tuple[int, int]:
    """Rows ``[lo, hi)`` owned by `rank` of `world` (row_blocks)."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    return row_blocks(b, world)[rank]


def aggregate_max(value: float, group=None, device=None) -> float:
    """Max of a per-rank scalar over the process group (job time = slowest rank).  Without an
    initialised process group, returns `value`."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def gather_rows(block: torch.Tensor, b: int, group=None) -> torch.Tensor:
    """All-gather the per-rank contiguous row blocks back into the full [B, ...] result (test and
    report helper; the truncation path itself never exchanges rows)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    blocks = row_blocks(b, world)
    width = max(hi - lo for lo, hi in blocks)
    pad = torch.zeros((width,) + tuple(block.shape[1:]), dtype=block.dtype, device=block.device)
    pad[:block.shape[0]] = block
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([parts[r][:hi - lo] for r, (lo, hi) in enumerate(blocks)], 0)


def _devices(devices: Optional[Sequence]) -> List[torch.device]:
    if devices is None:
        devices = list(range(torch.cuda.device_count()))
    devs = [torch.device("cuda", d) if isinstance(d, int) else torch.device(d) for d in devices]
    if not devs:
        raise ValueError("devices must name at least one CUDA device")
    for d in devs:
        if d.type != "cuda":
            raise ValueError(f"{d} is not a CUDA device")
        if d.index is None or d.index >= torch.cuda.device_count():
            raise ValueError(f"{d} is not available ({torch.cuda.device_count()} CUDA devices)")
    return devs


def _per_row_host(x, b: int, dtype, name: str) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        t = x.detach().to("cpu", dtype)
    else:
        t = torch.as_tensor(np.asarray(x), dtype=dtype)
    if t.dim() == 0:
        t = t.expand(b)
    if t.shape != (b,):
        raise ValueError(f"{name} must have shape ({b},), got {tuple(t.shape)}")
    return t.contiguous()


def topk_topp_sharded(logits, k, p, devices: Optional[Sequence] = None, *,
                      out: Optional[torch.Tensor] = None, flags: Optional[ops.TruncFlags] = None,
                      sample_size: int = ops.DEFAULT_SAMPLE_SIZE, check: bool = True,
                      kept_count: Optional[torch.Tensor] = None,
                      metrics: Optional[torch.Tensor] = None) -> torch.Tensor:
    """``topk_topp`` over contiguous row blocks on several devices (one block per entry of
    `devices`, default: every visible GPU).  Same result, bit for bit, as one ``topk_topp`` call.

    logits: host tensor / numpy array (masked logits come back in host memory, `out` if given), or a
    CUDA tensor (the result lands on the same device).  kept_count, if given, is an int32 [B] tensor
    on any device or the host; metrics (uint8 [B, 40], qrita_row_metrics) likewise.  check=True raises the reference's ValueError for
    invalid rows (row numbers are global)."""
    devs = _devices(devices)
    if isinstance(logits, np.ndarray):
        logits = torch.from_numpy(np.ascontiguousarray(logits))
    if not isinstance(logits, torch.Tensor):
        raise TypeError("logits must be a torch tensor or numpy array")
    if logits.dim() != 2:
        raise ValueError("logit batch must be 2-D (rows x vocab)")
    if logits.dtype not in ops._DTYPES:
        raise TypeError(f"unsupported dtype {logits.dtype}; expected float32 or bfloat16")
    b, v = logits.shape
    if b == 0 or v == 0:
        raise ValueError("batch_size and vocab_size must be >= 1")
    kh = _per_row_host(k, b, torch.int64, "k")
    ph = _per_row_host(p, b, torch.float64, "p")
    on_gpu = logits.is_cuda
    if not on_gpu:
        logits = logits.contiguous()
    if out is None:
        out = torch.empty_like(logits, pin_memory=(not on_gpu) and logits.is_pinned())
    elif out.shape != logits.shape or out.dtype != logits.dtype or out.device != logits.device or \
            not out.is_contiguous():
        raise ValueError("out must be a contiguous tensor matching logits (shape, dtype, device)")
    blocks = row_blocks(b, len(devs))
    counts: List[Optional[torch.Tensor]] = [None] * len(devs)
    mets: List[Optional[torch.Tensor]] = [None] * len(devs)
    errors: List[Optional[BaseException]] = [None] * len(devs)
    # the caller's stream on the input's device (thread-local in torch: captured here)
    src = torch.cuda.current_stream(logits.device) if on_gpu else None
    side = [ops.side_stream(d, i) if on_gpu and d == logits.device else None for i, d in enumerate(devs)]
    if on_gpu:
        for st in side:
            if st is not None:
                st.wait_stream(src)

    def work(i: int):
        lo, hi = blocks[i]
        if hi == lo:
            return
        dev = devs[i]
        try:
            ctx = torch.cuda.stream(side[i]) if side[i] is not None else contextlib.nullcontext()
            with torch.cuda.device(dev), ctx:
                kc = torch.empty(hi - lo, dtype=torch.int32, device=dev) if kept_count is not None else None
                mt = ops.metrics_buffer(hi - lo, dev) if metrics is not None else None
                if not on_gpu:
                    ops.topk_topp_host(logits[lo:hi], kh[lo:hi], ph[lo:hi], out=out[lo:hi], flags=flags,
                                       sample_size=sample_size, kept_count=kc, metrics=mt, check=check,
                                       device=dev, scratch_slot=i)
                elif side[i] is not None:
                    # same device: the block is a view; the result goes straight into out's rows
                    ops.topk_topp(logits[lo:hi], kh[lo:hi].to(dev, non_blocking=True),
                                  ph[lo:hi].to(dev, non_blocking=True), out=out[lo:hi], flags=flags,
                                  sample_size=sample_size, kept_count=kc, metrics=mt, check=check,
                                  stream=side[i])
                else:
                    # another device: peer copies (torch orders them against both devices' streams)
                    xb = logits[lo:hi].to(dev)
                    ob = ops.topk_topp(xb, kh[lo:hi].to(dev), ph[lo:hi].to(dev), flags=flags,
                                       sample_size=sample_size, kept_count=kc, metrics=mt, check=check)
                    out[lo:hi].copy_(ob.to(logits.device))
                    torch.cuda.current_stream(dev).synchronize()
                counts[i], mets[i] = kc, mt
                if side[i] is not None and (kc is not None or mt is not None):
                    side[i].synchronize()
        except BaseException as exc:  # re-raised in the caller's thread
            errors[i] = exc

    threads = [threading.Thread(target=work, args=(i,), daemon=True) for i in range(len(devs))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if on_gpu:
        for st in side:
            if st is not None:
                src.wait_stream(st)
    for exc in errors:
        if isinstance(exc, ops.TruncationError):
            # row numbers of the per-block check are local: report the batch's global rows
            raise ops.TruncationError("invalid batch: " + "; ".join(
                ops.describe_invalid(logits, kh, ph)[:5] or [str(exc)]))
    for exc in errors:
        if exc is not None:
            raise exc
    if kept_count is not None:
        for i, (lo, hi) in enumerate(blocks):
            if counts[i] is not None:
                kept_count[lo:hi].copy_(counts[i].to(kept_count.device))
    if metrics is not None:
        for i, (lo, hi) in enumerate(blocks):
            if mets[i] is not None:
                metrics[lo:hi].copy_(mets[i].to(metrics.device))
    return out
