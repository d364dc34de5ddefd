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
              check: Optional[bool] = None, stream: Optional[torch.cuda.Stream] = None,
              prep_event: Optional[torch.cuda.Event] = None,
              stream_event: Optional[torch.cuda.Event] = None) -> torch.Tensor:
    """Exact Top-k then Top-p truncation of a [B, V] tensor (fp32 or bf16) on the GPU.

    CUDA tensors are processed on their device, stream-ordered on `stream` (default: the current
    stream); the masked logits go to a new tensor, to `out`, or — with inplace=True — back into
    `logits` (which must then be row-contiguous: a tensor that would need a copy is rejected).  Host
    tensors go through topk_topp_host: row chunks are copied in, truncated and copied back with the
    transfers of both directions overlapped with the kernels (the result is a host tensor).

    k: int64 per row (k == V disables top-k); p: float64 per row (p == 1 disables top-p).  kept_count
    (int32 [B]) and metrics (uint8 [B, 40], qrita_row_metrics) are filled when given.

    check: raise the reference's ValueError for invalid rows (non-finite logits, k outside [1, V], p
    outside (0, 1]).  Checking SYNCHRONISES the stream and reads the device status block, so the
    default is check=False for CUDA tensors (the call stays fully asynchronous; invalid rows get
    undefined output) and check=True for host tensors (that call synchronises anyway).
    prep_event / stream_event (profiling only) are recorded after the preparation / streaming kernel;
    either one serialises the launches around it so the kernels can be timed alone.
    """
    if isinstance(logits, torch.Tensor) and not logits.is_cuda:
        if inplace or prep_event is not None or stream_event is not None:
            raise ValueError("host tensors support neither inplace nor profiling events")
        return topk_topp_host(logits, k, p, out=out, flags=flags, sample_size=sample_size,
                              kept_count=kept_count, metrics=metrics, check=True if check is None else check)
    if not isinstance(logits, torch.Tensor):
        raise TypeError("logits must be a torch tensor")
    if logits.dim() != 2:
        raise ValueError("logit batch must be 2-D (rows x vocab)")
    if logits.dtype not in _DTYPES:
        raise TypeError(f"unsupported dtype {logits.dtype}; expected float32 or bfloat16")
    if check is None:
        check = False
    if logits.stride(1) != 1 or (logits.shape[0] > 1 and logits.stride(0) < logits.shape[1]):
        if inplace:
            raise ValueError("inplace=True needs rows with unit column stride (this tensor would be copied)")
        logits = logits.contiguous()
    b, v = logits.shape
    if b == 0 or v == 0:
        raise ValueError("batch_size and vocab_size must be >= 1")
    if sample_size < 1:
        raise ValueError("sample_size must be >= 1")
    dev = logits.device
    st = stream or torch.cuda.current_stream(dev)
    if out is not None and not inplace and (out.shape != logits.shape or out.dtype != logits.dtype or
                                            out.stride(1) != 1):
        raise ValueError("out must match logits in shape/dtype with unit column stride")
    fl = (flags or TruncFlags()).bits() | (N.INPLACE if inplace else 0)
    lib = N.load()
    need = lib.qrita_workspace_bytes(b, v, _DTYPES[logits.dtype], fl)
    ws = workspace_for(dev, st)
    # temporaries (k / p in the kernel's dtypes, the output, the workspace) are created on the
    # launching stream, so the kernel never races their initialisation or their reuse
    with torch.cuda.device(dev), torch.cuda.stream(st):
        kt = _per_row(k, b, torch.int64, dev, "k")
        pt = _per_row(p, b, torch.float64, dev, "p")
        if inplace:
            out = logits
        elif out is None:
            out = torch.empty_like(logits)
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


def topk_topp_indices(logits: torch.Tensor, k: Union[int, torch.Tensor], p: Union[float, torch.Tensor], *,
                      kept_idx: Optional[torch.Tensor] = None, kept_count: Optional[torch.Tensor] = None,
                      out: Optional[torch.Tensor] = None, flags: Optional[TruncFlags] = None,
                      sample_size: int = DEFAULT_SAMPLE_SIZE, metrics: Optional[torch.Tensor] = None,
                      check: Optional[bool] = None, stream: Optional[torch.cuda.Stream] = None
                      ) -> Tuple[torch.Tensor, torch.Tensor]:
    """The kept columns of every row instead of (or besides, when `out` is given) the masked logits
    (qrita_topk_topp_idx; SURVEY.md 8b kept_idx).  Same selection as topk_topp.  Returns (kept_idx
    int32 [B, V], kept_count int32 [B]): row r's kept columns are kept_idx[r, :kept_count[r]], in
    unspecified order.  Without `out` only V * sizeof(dtype) is read and kept * 4 bytes written per
    row, about half of the masked-logit traffic.  CUDA tensors only; stream-ordered like topk_topp
    (check defaults to False: pass check=True to synchronise and raise for invalid rows)."""
    if not isinstance(logits, torch.Tensor) or not logits.is_cuda:
        raise TypeError("topk_topp_indices takes a CUDA tensor")
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
    if check is None:
        check = False
    if kept_idx is not None and (kept_idx.dtype != torch.int32 or kept_idx.dim() != 2 or
                                 kept_idx.shape[0] != b or kept_idx.shape[1] < v or kept_idx.stride(1) != 1):
        raise ValueError("kept_idx must be int32 [B, >= V] with unit column stride")
    if out is not None and (out.shape != logits.shape or out.dtype != logits.dtype or out.stride(1) != 1):
        raise ValueError("out must match logits in shape/dtype with unit column stride")
    fl = (flags or TruncFlags()).bits()
    st = stream or torch.cuda.current_stream(dev)
    lib = N.load()
    need = lib.qrita_workspace_bytes(b, v, _DTYPES[logits.dtype], fl)
    ws = workspace_for(dev, st)
    with torch.cuda.device(dev), torch.cuda.stream(st):
        kt = _per_row(k, b, torch.int64, dev, "k")
        pt = _per_row(p, b, torch.float64, dev, "p")
        if kept_idx is None:
            kept_idx = torch.empty((b, v), dtype=torch.int32, device=dev)
        if kept_count is None:
            kept_count = torch.empty((b,), dtype=torch.int32, device=dev)
        ws_ptr, ws_bytes = ws.get(need, st)
        rc = lib.qrita_topk_topp_idx(
            ctypes.c_void_p(logits.data_ptr()), _row_stride(logits), _DTYPES[logits.dtype], b, v,
            ctypes.c_void_p(kt.data_ptr()), ctypes.c_void_p(pt.data_ptr()),
            ctypes.c_void_p(out.data_ptr() if out is not None else 0), _row_stride(out) if out is not None else v,
            ctypes.c_void_p(kept_idx.data_ptr()), kept_idx.stride(0),
            ctypes.c_void_p(kept_count.data_ptr()),
            ctypes.c_void_p(metrics.data_ptr() if metrics is not None else 0),
            ctypes.c_void_p(ws_ptr), ws_bytes, fl, int(sample_size), ctypes.c_void_p(st.cuda_stream))
        if rc != N.OK:
            ws.reset()
            raise RuntimeError(f"qrita_topk_topp_idx failed: {N.strerror(rc)}")
        if check:
            check_status(ws_ptr, b, logits, kt, pt, st)
    return kept_idx, kept_count


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
# Host buffers: chunked, overlapped transfers (the pipeline itself is native: qrita_topk_topp_host)
# ------------------------------------------------------------------------------------------------
_host_lock = threading.Lock()
_host_scratch = {}
DEFAULT_HOST_CHUNK_BYTES = 16 << 20  # measured best on cfg2 (tools/e2e_sweep.py)


def _scratch_for(device: torch.device, nbytes: int, slot: int = 0) -> torch.Tensor:
    """Device scratch of the host-buffer pipeline per (device, slot), grown on demand (256-byte
    aligned).  Concurrent host-buffer calls on one device (topk_topp_sharded with a repeated device)
    use different slots."""
    with _host_lock:
        buf = _host_scratch.get((device.index, slot))
        if buf is None or buf.numel() < nbytes + 256:
            buf = torch.empty(nbytes + 256, dtype=torch.uint8, device=device)
            _host_scratch[(device.index, slot)] = buf
        return buf


_side_streams = {}


def side_stream(device: torch.device, slot: int) -> torch.cuda.Stream:
    """A library-owned CUDA stream per (device, slot) (row blocks of topk_topp_sharded)."""
    with _host_lock:
        st = _side_streams.get((device.index, slot))
        if st is None:
            st = torch.cuda.Stream(device=device)
            _side_streams[(device.index, slot)] = st
        return st


def topk_topp_host(logits: torch.Tensor, k, p, *, out: Optional[torch.Tensor] = None,
                   flags: Optional[TruncFlags] = None, sample_size: int = DEFAULT_SAMPLE_SIZE,
                   kept_count: Optional[torch.Tensor] = None, metrics: Optional[torch.Tensor] = None,
                   check: bool = True, device=None, chunk_bytes: int = DEFAULT_HOST_CHUNK_BYTES,
                   scratch_slot: int = 0) -> torch.Tensor:
    """topk_topp for a host [B, V] tensor through qrita_topk_topp_host: the library copies row chunks
    of ~chunk_bytes in, truncates each as soon as it has landed and copies it back, on three streams
    of its own, so both PCIe directions stay busy and overlap the kernels.  Pinned host memory gives
    asynchronous copies; pageable memory is staged through library-owned page-locked slots.  When
    every row is a top-k row (k < V, k <= 4096) only the kept columns come back and host threads
    build the masked rows from the input (bit-identical; not for a pageable input with a pinned out).
    Returns the masked logits as a host tensor (`out` when given); the call returns with the result in
    host memory.  kept_count / metrics, if given, are CUDA tensors.  check=True raises the
    reference's ValueError for invalid rows."""
    if logits.dim() != 2:
        raise ValueError("logit batch must be 2-D (rows x vocab)")
    if logits.dtype not in _DTYPES:
        raise TypeError(f"unsupported dtype {logits.dtype}; expected float32 or bfloat16")
    logits = logits.contiguous()
    b, v = logits.shape
    if b == 0 or v == 0:
        raise ValueError("batch_size and vocab_size must be >= 1")
    if sample_size < 1:
        raise ValueError("sample_size must be >= 1")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if out is None:
        out = torch.empty_like(logits, pin_memory=logits.is_pinned())
    elif out.shape != logits.shape or out.dtype != logits.dtype or out.is_cuda or not out.is_contiguous():
        raise ValueError("out must be a contiguous host tensor matching logits")
    cpu = torch.device("cpu")
    kt = _per_row(k, b, torch.int64, cpu, "k")
    pt = _per_row(p, b, torch.float64, cpu, "p")
    for t, nm in ((kept_count, "kept_count"), (metrics, "metrics")):
        if t is not None and (not t.is_cuda or t.device != dev or not t.is_contiguous()):
            raise ValueError(f"{nm} must be a contiguous CUDA tensor on {dev}")
    lib = N.load()
    dt = _DTYPES[logits.dtype]
    fl = (flags or TruncFlags()).bits()
    rows = max(1, min(b, chunk_bytes // (v * logits.element_size())))
    need = lib.qrita_host_scratch_bytes(b, v, dt, rows)
    with torch.cuda.device(dev):
        st = torch.cuda.current_stream(dev)
        buf = _scratch_for(dev, need, scratch_slot)
        base = buf.data_ptr()
        sp = (base + 255) & ~255
        rc = lib.qrita_topk_topp_host(
            ctypes.c_void_p(logits.data_ptr()), dt, b, v, ctypes.c_void_p(kt.data_ptr()),
            ctypes.c_void_p(pt.data_ptr()), ctypes.c_void_p(out.data_ptr()),
            ctypes.c_void_p(kept_count.data_ptr() if kept_count is not None else 0),
            ctypes.c_void_p(metrics.data_ptr() if metrics is not None else 0),
            ctypes.c_void_p(sp), buf.numel() - (sp - base), rows, fl, int(sample_size),
            ctypes.c_void_p(st.cuda_stream))
        if rc != N.OK:
            raise RuntimeError(f"qrita_topk_topp_host failed: {N.strerror(rc)}")
        if check:
            row, col = ctypes.c_int(-1), ctypes.c_int(-1)
            code = lib.qrita_get_status_host(ctypes.c_void_p(sp), b, v, dt, rows, ctypes.byref(row),
                                             ctypes.byref(col), ctypes.c_void_p(st.cuda_stream))
            if code in (N.ENONFINITE, N.EINVAL_K, N.EINVAL_P):
                raise TruncationError("invalid batch: " + "; ".join(
                    describe_invalid(logits, kt, pt)[:5] or [N.strerror(code)]))
            if code != N.OK:
                raise RuntimeError(f"qrita_get_status_host failed: {N.strerror(code)}")
        st.synchronize()
    return out
