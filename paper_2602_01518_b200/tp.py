"""Vocab-sharded (tensor-parallel LM-head) exact Top-k / Top-p — BASELINE config cfg5, SURVEY.md §8e.

Each rank holds a contiguous column shard ``[B, V_r]`` of the logits (columns
``[offset_r, offset_r + V_r)``, offsets increasing with rank) and receives its shard of the
*unsharded* answer (oracle.py:70-89; pipeline.py:199-239), bit-exact.

The protocol is native (``qrita_topk_topp_tp`` in libqrita_b200.so, csrc/qrita_tp.cu): local top-k
candidates -> one all-gather of (order key, global column) pairs -> the exact resolve on the
gathered candidates; rows that are top-p only (k == V) exchange only exact fixed-point mass
partials (integer all-reduce SUM) of a radix search for the nucleus boundary plus the per-rank
boundary-tie counts.  No logits cross ranks.

The exchange goes through a communicator object:

* ``NcclComm(group)`` — a library-owned NCCL communicator over the ranks of a torch process group
  (the unique id travels through ``torch.distributed``); collectives run on the GPU, stream-ordered.
* ``TorchComm(group)`` — host-staged collectives through ``torch.distributed`` (any backend, e.g.
  gloo): the device buffer is copied to the host, reduced / gathered, copied back.
* ``ThreadComm`` — ranks as threads of one process (each with its own CUDA stream), exchanging
  through host memory: ``simulate_tp`` runs the real multi-rank protocol on one GPU.
"""
from __future__ import annotations

import ctypes
import threading
from typing import List, Optional

import numpy as np
import torch

from . import _native as N
from . import ops

_ALLREDUCE = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p,
                              ctypes.c_void_p)
_ALLGATHER = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p,
                              ctypes.c_void_p)


class QritaComm(ctypes.Structure):
    """qrita_comm (include/qrita_b200.h)."""

    _fields_ = [("all_reduce_sum", _ALLREDUCE), ("all_gather", _ALLGATHER), ("ctx", ctypes.c_void_p)]


class _HostStagedComm:
    """Common part of the host-staged communicators: device <-> host copies around a host
    collective `_reduce(np.ndarray) -> np.ndarray` / `_gather(np.ndarray) -> List[np.ndarray]`."""

    def __init__(self):
        self._cb = QritaComm(_ALLREDUCE(self._all_reduce_sum), _ALLGATHER(self._all_gather), None)
        self.bytes_exchanged = 0   # payload bytes this rank sent, for reports

    @property
    def c(self) -> QritaComm:
        return self._cb

    def _d2h(self, ptr: int, nbytes: int, stream: int) -> np.ndarray:
        host = np.empty(nbytes, dtype=np.uint8)
        if N.load().qrita_copy_sync(host.ctypes.data, ptr, nbytes, stream) != N.OK:
            raise RuntimeError("device -> host copy failed")
        return host

    def _h2d(self, ptr: int, host: np.ndarray, stream: int):
        host = np.ascontiguousarray(host)
        if N.load().qrita_copy_sync(ptr, host.ctypes.data, host.nbytes, stream) != N.OK:
            raise RuntimeError("host -> device copy failed")

    def _all_reduce_sum(self, buf, count, elem_bytes, stream, ctx):
        try:
            dt = np.uint64 if elem_bytes == 8 else np.uint32
            host = self._d2h(buf, count * elem_bytes, stream).view(dt)
            self.bytes_exchanged += host.nbytes
            self._h2d(buf, self._reduce(host), stream)
            return 0
        except Exception as exc:  # reported as QRITA_ENCCL by the library
            self.error = exc
            return 1

    def _all_gather(self, send, recv, nbytes, stream, ctx):
        try:
            host = self._d2h(send, nbytes, stream)
            self.bytes_exchanged += host.nbytes
            self._h2d(recv, np.concatenate(self._gather(host)), stream)
            return 0
        except Exception as exc:
            self.error = exc
            return 1


class TorchComm(_HostStagedComm):
    """Host-staged collectives over a torch.distributed process group (gloo in the CPU-side tests;
    any backend works)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        super().__init__()
        self.dist, self.group = dist, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def _reduce(self, host: np.ndarray) -> np.ndarray:
        t = torch.from_numpy(host.view(np.int64 if host.dtype == np.uint64 else np.int32).copy())
        self.dist.all_reduce(t, group=self.group)   # two's-complement sums wrap like unsigned ones
        return t.numpy().view(host.dtype)

    def _gather(self, host: np.ndarray) -> List[np.ndarray]:
        t = torch.from_numpy(host)
        parts = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(parts, t, group=self.group)
        return [p.numpy() for p in parts]


class ThreadGroup:
    """Ranks as threads of one process (simulate_tp): a barrier and one host slot per rank."""

    def __init__(self, world: int):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots: List[Optional[np.ndarray]] = [None] * world


class ThreadComm(_HostStagedComm):
    def __init__(self, group: ThreadGroup, rank: int):
        super().__init__()
        self.g, self.rank, self.world = group, rank, group.world

    def _exchange(self, host: np.ndarray) -> List[np.ndarray]:
        self.g.slots[self.rank] = host
        self.g.barrier.wait()
        parts = list(self.g.slots)
        self.g.barrier.wait()   # every rank has read every slot before they are reused
        return parts

    def _reduce(self, host: np.ndarray) -> np.ndarray:
        parts = self._exchange(host)
        out = parts[0].copy()
        for q in parts[1:]:
            out += q            # unsigned wrap-around, like the integer collectives
        return out

    def _gather(self, host: np.ndarray) -> List[np.ndarray]:
        return self._exchange(host)


class NcclComm:
    """A library-owned NCCL communicator over the ranks of a torch.distributed group: rank 0 draws
    the unique id (qrita_nccl_unique_id), the group broadcasts it, every rank joins on its current
    CUDA device (qrita_nccl_comm_init).  Collectives are enqueued on the call's stream."""

    def __init__(self, group=None):
        import torch.distributed as dist
        lib = N.load()
        single = not (dist.is_available() and dist.is_initialized())   # one rank, no process group
        self.rank, self.world = (0, 1) if single else (dist.get_rank(group), dist.get_world_size(group))
        uid = ctypes.create_string_buffer(128)
        if self.rank == 0 and lib.qrita_nccl_unique_id(uid) != N.OK:
            raise RuntimeError("qrita_nccl_unique_id failed (is libnccl.so.2 loadable?)")
        obj = [uid.raw]
        if not single:
            src = dist.get_global_rank(group, 0) if group is not None else 0
            dist.broadcast_object_list(obj, src=src, group=group)
        self.handle = ctypes.c_void_p()
        if lib.qrita_nccl_comm_init(ctypes.byref(self.handle), self.world, obj[0], self.rank) != N.OK:
            raise RuntimeError("qrita_nccl_comm_init failed")

    def close(self):
        if self.handle:
            N.load().qrita_nccl_comm_destroy(self.handle)
            self.handle = ctypes.c_void_p()


_ws_lock = threading.Lock()
_tp_ws = {}


def _workspace(dev: torch.device, stream: torch.cuda.Stream, nbytes: int) -> tuple:
    key = (dev.index, stream.cuda_stream)
    with _ws_lock:
        buf = _tp_ws.get(key)
        if buf is None or buf.numel() < nbytes + 256:
            buf = torch.zeros(nbytes + 256, dtype=torch.uint8, device=dev)   # zeroed before first use
            _tp_ws[key] = buf
    base = buf.data_ptr()
    aligned = (base + 255) & ~255
    return aligned, buf.numel() - (aligned - base), buf


def topk_topp_tp(shard: torch.Tensor, k, p, *, vocab_offset: int, vocab_size: int, comm=None,
                 rank: Optional[int] = None, world: Optional[int] = None, k_cap: Optional[int] = None,
                 out: Optional[torch.Tensor] = None, inplace: bool = False,
                 kept_count: Optional[torch.Tensor] = None, check: bool = False,
                 stream: Optional[torch.cuda.Stream] = None, topp_only_rows: Optional[bool] = None) -> torch.Tensor:
    """Exact truncation of a vocab shard [B, V_r] (CUDA, fp32 or bf16): this rank's shard of the
    global answer.  k (int64) / p (float64) are the GLOBAL per-row targets.  comm: NcclComm,
    TorchComm, ThreadComm (default: NcclComm over the default group when its backend is NCCL, else
    TorchComm).  k_cap bounds every k < vocab_size (default: computed from k, one sync).  kept_count
    receives the entries kept in this shard.  topp_only_rows: whether some row is top-p only
    (k == vocab_size, p < 1); False skips the top-p rounds (default: computed from k / p, one sync).
    check=True synchronises and raises the reference's ValueError for invalid rows of this shard."""
    if not isinstance(shard, torch.Tensor) or not shard.is_cuda or shard.dim() != 2:
        raise TypeError("shard must be a 2-D CUDA tensor")
    if shard.dtype not in ops._DTYPES:
        raise TypeError(f"unsupported dtype {shard.dtype}; expected float32 or bfloat16")
    if shard.stride(1) != 1:
        if inplace:
            raise ValueError("inplace=True needs a shard with unit column stride")
        shard = shard.contiguous()
    b, vr = shard.shape
    dev = shard.device
    st = stream or torch.cuda.current_stream(dev)
    if comm is None:
        import torch.distributed as dist
        comm = _default_comm()
        rank, world = dist.get_rank(), dist.get_world_size()
    if rank is None:
        rank = comm.rank
    if world is None:
        world = comm.world
    with torch.cuda.device(dev), torch.cuda.stream(st):
        kt = ops._per_row(k, b, torch.int64, dev, "k")
        pt = ops._per_row(p, b, torch.float64, dev, "p")
        if k_cap is None:
            small = kt[kt < vocab_size]
            k_cap = int(small.max().item()) if small.numel() else 1
        if topp_only_rows is None:
            topp_only_rows = bool(((kt >= vocab_size) & (pt < 1.0)).any().item())
        no_topp = not topp_only_rows
        if inplace:
            out = shard
        elif out is None:
            out = torch.empty_like(shard)
        elif out.shape != shard.shape or out.dtype != shard.dtype or out.stride(1) != 1:
            raise ValueError("out must match the shard in shape/dtype with unit column stride")
        lib = N.load()
        dt = ops._DTYPES[shard.dtype]
        need = lib.qrita_tp_workspace_bytes(b, vr, dt, world, int(k_cap))
        ws_ptr, ws_bytes, _keep = _workspace(dev, st, need)
        fl = (N.INPLACE if inplace else 0) | (N.TP_NO_TOPP_ROWS if no_topp else 0)
        args = (ctypes.c_void_p(shard.data_ptr()), ops._row_stride(shard), dt, b, vr, int(vocab_size),
                int(vocab_offset), ctypes.c_void_p(kt.data_ptr()), ctypes.c_void_p(pt.data_ptr()), int(k_cap),
                ctypes.c_void_p(out.data_ptr()), ops._row_stride(out),
                ctypes.c_void_p(kept_count.data_ptr() if kept_count is not None else 0),
                ctypes.c_void_p(ws_ptr), ws_bytes, fl, int(rank), int(world))
        if isinstance(comm, NcclComm):
            rc = lib.qrita_topk_topp_tp(*args, comm.handle, ctypes.c_void_p(st.cuda_stream))
        else:
            rc = lib.qrita_topk_topp_tp_comm(*args, ctypes.c_void_p(ctypes.addressof(comm.c)),
                                             ctypes.c_void_p(st.cuda_stream))
        if rc != N.OK:
            err = getattr(comm, "error", None)
            raise RuntimeError(f"qrita_topk_topp_tp failed: {N.strerror(rc)}" + (f" ({err!r})" if err else ""))
        if check:
            ops.check_status(ws_ptr, b, shard, kt, pt, st)
    return out


_default = {}


def _default_comm():
    import torch.distributed as dist
    key = id(dist.group.WORLD)
    c = _default.get(key)
    if c is None:
        c = NcclComm() if dist.get_backend() == "nccl" else TorchComm()
        _default[key] = c
    return c


def shard_bounds(v: int, world: int) -> List[int]:
    """Column offsets of `world` contiguous shards of a V-column row (shard r = [b[r], b[r+1]))."""
    return [v * r // world for r in range(world + 1)]


def simulate_tp(x: torch.Tensor, k, p, world: int, k_cap: Optional[int] = None,
                kept_count: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Run the native TP protocol for `world` column shards of x inside one process: one thread and
    one CUDA stream per rank, exchanging through host memory (ThreadComm).  Returns the full masked
    matrix (the concatenated shard outputs); kept_count (int32 [B], optional) sums the shards."""
    b, v = x.shape
    dev = x.device
    bounds = shard_bounds(v, world)
    group = ThreadGroup(world)
    outs: List[Optional[torch.Tensor]] = [None] * world
    kcs: List[Optional[torch.Tensor]] = [None] * world
    errs: List[Optional[BaseException]] = [None] * world
    kt = ops._per_row(k, b, torch.int64, dev, "k")
    pt = ops._per_row(p, b, torch.float64, dev, "p")
    if k_cap is None:
        small = kt[kt < v]
        k_cap = int(small.max().item()) if small.numel() else 1
    torch.cuda.synchronize(dev)

    def rank_fn(r: int):
        try:
            st = ops.side_stream(dev, 1000 + r)
            with torch.cuda.device(dev), torch.cuda.stream(st):
                shard = x[:, bounds[r]:bounds[r + 1]].contiguous()
                kc = torch.zeros(b, dtype=torch.int32, device=dev)
                outs[r] = topk_topp_tp(shard, kt, pt, vocab_offset=bounds[r], vocab_size=v,
                                       comm=ThreadComm(group, r), k_cap=k_cap, kept_count=kc, stream=st)
                kcs[r] = kc
                st.synchronize()
        except BaseException as exc:
            errs[r] = exc
            group.barrier.abort()

    threads = [threading.Thread(target=rank_fn, args=(r,), daemon=True) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for e in errs:
        if e is not None and not isinstance(e, threading.BrokenBarrierError):
            raise e
    for e in errs:
        if e is not None:
            raise e
    if kept_count is not None:
        kept_count.copy_(torch.stack(kcs).sum(0).to(kept_count.dtype))
    return torch.cat(outs, dim=1)
