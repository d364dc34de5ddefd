"""Device-level operator: exact Top-k / Top-p truncation of CUDA logit tensors.

This is the stream-ordered call that every public entry point (engine.run_batch, the per-row
pipeline functions, the vocab-sharded variant, bench.py) goes through.  It hands raw device pointers
to `qrita_topk_topp` in libqrita_b200.so (include/qrita_b200.h).  PyTorch is used only for device
memory and the current stream.  There is no CPU path: CPU tensors are rejected.
"""
from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass
from typing import Optional, Tuple, Union

import torch

from . import _native as N

DEFAULT_SAMPLE_SIZE = 4096  # sigma_trunc.py:21

_DTYPES = {torch.float32: N.DTYPE_F32, torch.bfloat16: N.DTYPE_BF16}


@dataclass
class TruncFlags:
    """The reference's EngineConfig ablation switches (engine.py:26-40) as kernel flags."""

    search: str = "quaternary"          # or "binary"
    use_sigma_trunc: bool = True
    force_fallback: bool = False
    dup_handling: bool = True
    debug_timing: bool = False          # record tail phase timestamps (qrita_get_timing)
    staged: bool = False                # force the staged prep/stream/tail pipeline (ablation)

    def bits(self) -> int:
        if self.search not in ("quaternary", "binary"):
            raise ValueError("search_kind must be 'quaternary' or 'binary'")
        f = 0
        if self.search == "binary":
            f |= N.SEARCH_BINARY
        if not self.use_sigma_trunc:
            f |= N.NO_SIGMA
        if self.force_fallback:
            f |= N.FORCE_FALLBACK
        if not self.dup_handling:
            f |= N.NO_DUP
        if self.debug_timing:
            f |= N.DEBUG_TIMING
        if self.staged:
            f |= N.STAGED
        return f


class Workspace:
    """Device scratch for one stream: grown on demand, zeroed once; every call leaves it clean."""

    def __init__(self, device: torch.device):
        self.device = device
        self.buf: Optional[torch.Tensor] = None

    def get(self, nbytes: int, stream: torch.cuda.Stream) -> Tuple[int, int]:
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = None
            self.buf = torch.zeros(max(nbytes, 1 << 20) + 256, dtype=torch.uint8, device=self.device)
        ptr = self.buf.data_ptr()
        aligned = (ptr + 255) & ~255
        return aligned, self.buf.numel() - (aligned - ptr)

    def reset(self):
        if self.buf is not None:
            self.buf.zero_()


_ws_lock = threading.Lock()
_workspaces = {}


def workspace_for(device: torch.device, stream: torch.cuda.Stream) -> Workspace:
    key = (device.index, stream.cuda_stream)
    with _ws_lock:
        ws = _workspaces.get(key)
        if ws is None:
            ws = Workspace(device)
            _workspaces[key] = ws
        return ws


def _per_row(x, b: int, dtype: torch.dtype, device: torch.device, name: str) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        t = x.to(device=device, dtype=dtype)
        if t.dim() == 0:
            t = t.expand(b)
        if t.shape != (b,):
            raise ValueError(f"{name} must have shape ({b},), got {tuple(t.shape)}")
        return t.contiguous()
    return torch.full((b,), x, dtype=dtype, device=device)


def _row_stride(t: torch.Tensor) -> int:
    # a size-1 batch dimension may carry any stride (numpy/torch relaxed strides)
    return t.stride(0) if t.shape[0] > 1 else t.shape[1]


class TruncationError(ValueError):
    """Raised with the reference's ValueError wording (core.py:126-139)."""


def check_status(ws_ptr: int, b: int, logits: Optional[torch.Tensor], k, p,
                 stream: torch.cuda.Stream) -> None:
    """Synchronise and translate the device status block into the reference's ValueError."""
    lib = N.load()
    row, col = ctypes.c_int(-1), ctypes.c_int(-1)
    code = lib.qrita_get_status(ctypes.c_void_p(ws_ptr), b, ctypes.byref(row), ctypes.byref(col),
                                ctypes.c_void_p(stream.cuda_stream))
    if code == N.OK:
        return
    if code in (N.ENONFINITE, N.EINVAL_K, N.EINVAL_P):
        raise TruncationError("invalid batch: " + "; ".join(
            describe_invalid(logits, k, p)[:5] or [N.strerror(code)]))
    raise RuntimeError(f"qrita_get_status failed: {N.strerror(code)}")


def describe_invalid(logits: Optional[torch.Tensor], k, p) -> list:
    """validate_batch's report lines (core.py:120-140), computed on the device tensors."""
    report = []
    if logits is not None:
        bad = ~torch.isfinite(logits)
        if bool(bad.any()):
            for r, c in torch.nonzero(bad)[:5].tolist():
                kind = "NaN" if bool(torch.isnan(logits[r, c])) else "non-finite"
                report.append(f"{kind} logit at row {r}, col {c}")
    v = logits.shape[1] if logits is not None else None
    if isinstance(k, torch.Tensor) and v is not None:
        for r, kk in enumerate(k.tolist()):
            if not (1 <= kk <= v):
                report.append(f"row {r}: k out of range [1,V] (k={kk}, V={v})")
    if isinstance(p, torch.Tensor):
        for r, pp in enumerate(p.tolist()):
            if not (0.0 < pp <= 1.0):
                report.append(f"row {r}: p out of range (0,1] (p={pp})")
    return report


def topk_topp(logits: torch.Tensor, k: Union[int, torch.Tensor], p: Union[float, torch.Tensor], *,
              out: Optional[torch.Tensor] = None, inplace: bool = False,
              flags: Optional[TruncFlags] = None, sample_size: int = DEFAULT_SAMPLE_SIZE,
              kept_count: Optional[torch.Tensor] = None, metrics: Optional[torch.Tensor] = None,
              check: bool = True, stream: Optional[torch.cuda.Stream] = None,
              prep_event: Optional[torch.cuda.Event] = None,
              stream_event: Optional[torch.cuda.Event] = None) -> torch.Tensor:
    """Exact Top-k then Top-p truncation of a [B, V] tensor (fp32 or bf16) on the GPU.

    CUDA tensors are truncated in place on their device (stream-ordered).  Host tensors go through
    topk_topp_host: row chunks are copied in, truncated and copied back with the transfers of both
    directions overlapped with the kernels (the result is a host tensor).

    k: int64 per row (k == V disables top-k); p: float64 per row (p == 1 disables top-p).  Returns
    the masked logits (new tensor, or `logits` itself when inplace).  kept_count (int32 [B]) and
    metrics (uint8 [B, 40], qrita_row_metrics) are filled when given.  check=True synchronises and
    raises the reference's ValueError for invalid rows; check=False leaves the call fully async.
    prep_event / stream_event (profiling only) are recorded after the preparation / streaming kernel;
    either one serialises the launches around it so the kernels can be timed alone.
    """
    if isinstance(logits, torch.Tensor) and not logits.is_cuda:
        if inplace or prep_event is not None or stream_event is not None:
            raise ValueError("host tensors support neither inplace nor profiling events")
        return topk_topp_host(logits, k, p, out=out, flags=flags, sample_size=sample_size,
                              kept_count=kept_count, metrics=metrics, check=check)
    if not isinstance(logits, torch.Tensor):
        raise TypeError("logits must be a torch tensor")
    if logits.dim() != 2:
        raise ValueError("logit batch must be 2-D (rows x vocab)")
    if logits.dtype not in _DTYPES:
        raise TypeError(f"unsupported dtype {logits.dtype}; expected float32 or bfloat16")
    if logits.stride(1) != 1 or (logits.shape[0] > 1 and logits.stride(0) < logits.shape[1]):
        logits = logits.contiguous()
    b, v = logits.shape
    if b == 0 or v == 0:
        raise ValueError("batch_size and vocab_size must be >= 1")
    if sample_size < 1:
        raise ValueError("sample_size must be >= 1")
    dev = logits.device
    kt = _per_row(k, b, torch.int64, dev, "k")
    pt = _per_row(p, b, torch.float64, dev, "p")
    if inplace:
        out = logits
    elif out is None:
        out = torch.empty_like(logits)
    elif out.shape != logits.shape or out.dtype != logits.dtype or out.stride(1) != 1:
        raise ValueError("out must match logits in shape/dtype with unit column stride")
    fl = (flags or TruncFlags()).bits() | (N.INPLACE if inplace else 0)
    st = stream or torch.cuda.current_stream(dev)
    lib = N.load()
    need = lib.qrita_workspace_bytes(b, v, _DTYPES[logits.dtype], fl)
    ws = workspace_for(dev, st)
    with torch.cuda.device(dev):
        ws_ptr, ws_bytes = ws.get(need, st)
        ev = ev2 = 0
        if prep_event is not None:
            prep_event.record(st)  # materialise the event handle, re-recorded by the library
            ev = prep_event.cuda_event
        if stream_event is not None:
            stream_event.record(st)
            ev2 = stream_event.cuda_event
        rc = lib.qrita_topk_topp_ex(
            ctypes.c_void_p(logits.data_ptr()), _row_stride(logits), _DTYPES[logits.dtype], b, v,
            ctypes.c_void_p(kt.data_ptr()), ctypes.c_void_p(pt.data_ptr()),
            ctypes.c_void_p(out.data_ptr()), _row_stride(out),
            ctypes.c_void_p(kept_count.data_ptr() if kept_count is not None else 0),
            ctypes.c_void_p(metrics.data_ptr() if metrics is not None else 0),
            ctypes.c_void_p(ws_ptr), ws_bytes, fl, int(sample_size),
            ctypes.c_void_p(st.cuda_stream), ctypes.c_void_p(ev), ctypes.c_void_p(ev2))
        if rc != N.OK:
            ws.reset()
            raise RuntimeError(f"qrita_topk_topp failed: {N.strerror(rc)}")
        if check:
            check_status(ws_ptr, b, logits, kt, pt, st)
    return out


def pipeline_kind(logits: torch.Tensor, flags: Optional[TruncFlags] = None) -> str:
    """Which kernel pipeline qrita_topk_topp runs for this tensor (mirrors the dispatch in
    csrc/qrita_impl.cuh launch_all): "fused" (one launch: qrita_fused) when rows are 16-byte aligned
    for the bulk copies, else "staged" (qrita_prep -> qrita_stream -> qrita_tail)."""
    es = logits.element_size()
    v = logits.shape[1]
    ld = _row_stride(logits)
    aligned = logits.data_ptr() % 16 == 0 and (ld * es) % 16 == 0 and (v * es) % 16 == 0
    staged = flags is not None and flags.staged
    return "fused" if aligned and not staged else "staged"


def metrics_buffer(b: int, device) -> torch.Tensor:
    return torch.zeros((b, N.METRICS_BYTES), dtype=torch.uint8, device=device)


def decode_metrics(buf: torch.Tensor):
    """uint8 [B, 40] qrita_row_metrics -> list of dicts (host)."""
    raw = buf.cpu().numpy().tobytes()
    rows = []
    sz = N.METRICS_BYTES
    for i in range(buf.shape[0]):
        m = N.RowMetricsC.from_buffer_copy(raw[i * sz:(i + 1) * sz])
        rows.append({f: getattr(m, f) for f, _ in N.RowMetricsC._fields_})
    return rows


# ------------------------------------------------------------------------------------------------
# Host buffers: chunked, overlapped transfers
# ------------------------------------------------------------------------------------------------
_host_lock = threading.Lock()
_host_streams = {}


def _streams_for(device: torch.device, n: int):
    key = (device.index, n)
    with _host_lock:
        ss = _host_streams.get(key)
        if ss is None:
            ss = [torch.cuda.Stream(device) for _ in range(n)]
            _host_streams[key] = ss
        return ss


def _status_view(ws: Workspace, b: int) -> torch.Tensor:
    """The [status[b] | nf_col[b]] words at the head of a workspace (include/qrita_b200.h layout)."""
    base = ws.buf.data_ptr()
    off = ((base + 255) & ~255) - base
    nf_off = off + ((4 * b + 255) // 256) * 256
    st = ws.buf[off:off + 4 * b].view(torch.int32)
    nf = ws.buf[nf_off:nf_off + 4 * b].view(torch.int32)
    return st, nf


def topk_topp_host(logits: torch.Tensor, k, p, *, out: Optional[torch.Tensor] = None,
                   flags: Optional[TruncFlags] = None, sample_size: int = DEFAULT_SAMPLE_SIZE,
                   kept_count: Optional[torch.Tensor] = None, metrics: Optional[torch.Tensor] = None,
                   check: bool = True, device=None, chunk_bytes: int = 16 << 20) -> torch.Tensor:
    """topk_topp for a host [B, V] tensor.  Three streams: one uploads row chunks of ~chunk_bytes back
    to back, one truncates each chunk as soon as it has landed, one downloads each result as soon
    as it is ready, so both PCIe directions stay busy and overlap the kernels (per-chunk events
    order them).  Pinned host memory gives asynchronous copies; pageable memory works, synchronously.
    Returns the masked logits as a host tensor (`out` when given).  kept_count / metrics, if given,
    are CUDA tensors.  check=True raises the reference's ValueError for invalid rows (after all
    chunks ran); the call always returns with the result in host memory."""
    if logits.dim() != 2:
        raise ValueError("logit batch must be 2-D (rows x vocab)")
    if logits.dtype not in _DTYPES:
        raise TypeError(f"unsupported dtype {logits.dtype}; expected float32 or bfloat16")
    logits = logits.contiguous()
    b, v = logits.shape
    if b == 0 or v == 0:
        raise ValueError("batch_size and vocab_size must be >= 1")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if out is None:
        out = torch.empty_like(logits, pin_memory=logits.is_pinned())
    elif out.shape != logits.shape or out.dtype != logits.dtype or out.is_cuda or not out.is_contiguous():
        raise ValueError("out must be a contiguous host tensor matching logits")
    kt = _per_row(k, b, torch.int64, dev, "k")
    pt = _per_row(p, b, torch.float64, dev, "p")
    up, comp, down = _streams_for(dev, 3)
    cur = torch.cuda.current_stream(dev)
    status = torch.zeros((b,), dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        xd = torch.empty((b, v), dtype=logits.dtype, device=dev)
        od = torch.empty((b, v), dtype=logits.dtype, device=dev)
        for s in (up, comp, down):
            s.wait_stream(cur)  # k / p / status / buffers were produced on the current stream
        rows = max(1, min(b, chunk_bytes // (v * logits.element_size())))
        spans = [(r0, min(b, r0 + rows)) for r0 in range(0, b, rows)]
        landed, done = [], []
        with torch.cuda.stream(up):
            for r0, r1 in spans:
                xd[r0:r1].copy_(logits[r0:r1], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(up)
                landed.append(ev)
        with torch.cuda.stream(comp):
            # lean per-chunk launches straight through the C ABI (arguments prepared once)
            lib = N.load()
            dt = _DTYPES[logits.dtype]
            fl = (flags or TruncFlags()).bits()
            esz = logits.element_size()
            maxr = max(r1 - r0 for r0, r1 in spans)
            ws = workspace_for(dev, comp)
            ws_ptr, ws_bytes = ws.get(lib.qrita_workspace_bytes(maxr, v, dt, fl), comp)
            st_all, _ = _status_view(ws, maxr)
            x0, o0, k0, p0 = xd.data_ptr(), od.data_ptr(), kt.data_ptr(), pt.data_ptr()
            kc0 = kept_count.data_ptr() if kept_count is not None else 0
            me0 = metrics.data_ptr() if metrics is not None else 0
            cs = ctypes.c_void_p(comp.cuda_stream)
            for (r0, r1), ev in zip(spans, landed):
                comp.wait_event(ev)
                rc = lib.qrita_topk_topp(
                    ctypes.c_void_p(x0 + r0 * v * esz), v, dt, r1 - r0, v,
                    ctypes.c_void_p(k0 + 8 * r0), ctypes.c_void_p(p0 + 8 * r0),
                    ctypes.c_void_p(o0 + r0 * v * esz), v,
                    ctypes.c_void_p(kc0 + 4 * r0 if kc0 else 0),
                    ctypes.c_void_p(me0 + N.METRICS_BYTES * r0 if me0 else 0),
                    ctypes.c_void_p(ws_ptr), ws_bytes, fl, int(sample_size), cs)
                if rc != N.OK:
                    raise RuntimeError(f"qrita_topk_topp failed: {N.strerror(rc)}")
                status[r0:r1].copy_(st_all[:r1 - r0], non_blocking=True)
                ev2 = torch.cuda.Event()
                ev2.record(comp)
                done.append(ev2)
        with torch.cuda.stream(down):
            for (r0, r1), ev in zip(spans, done):
                down.wait_event(ev)
                out[r0:r1].copy_(od[r0:r1], non_blocking=True)
        for s in (up, comp, down):
            cur.wait_stream(s)
        for t in (xd, od, status):
            for s in (up, comp, down):
                t.record_stream(s)
        if check:
            if bool(status.ne(0).any()):  # synchronises
                raise TruncationError("invalid batch: " + "; ".join(
                    describe_invalid(logits, kt.cpu(), pt.cpu())[:5] or ["invalid rows"]))
        torch.cuda.synchronize(dev)
    return out
