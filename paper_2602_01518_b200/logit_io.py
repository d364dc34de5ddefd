"""QRTL logit files and per-row target CSVs — the reference's logit_io.py format (pkg/src/sigmatop/
logit_io.py:16-72), byte-compatible in both directions, plus direct paths to and from the GPU.

Layout: 16-byte little-endian header (magic "QRTL", u32 version = 1, u32 B, u32 V) followed by
B*V float32 values row-major.  Masked outputs use the same format (-inf is representable on disk;
input validation rejects it).

Beyond the reference: ``read_logits(path, device="cuda")`` lands the payload in HBM through a
page-locked staging buffer (no intermediate numpy copy), and ``write_logits`` accepts CUDA tensors
and bf16 logits (upcast to fp32, exact), so real-model logits (e.g. an LM head's output tensor)
can be cached as QRTL and replayed through run_batch / bench / verify.
"""
from __future__ import annotations

import csv
import os
import struct

import numpy as np
import torch

from .core import LogitBatch, TruncTargets, _is_tensor

MAGIC = b"QRTL"
VERSION = 1
_HEADER = struct.Struct("<4sIII")


def _read_header(fh, path):
    header = fh.read(_HEADER.size)
    if len(header) != _HEADER.size:
        raise ValueError(f"{path}: truncated header")
    magic, version, b, v = _HEADER.unpack(header)
    if magic != MAGIC:
        raise ValueError(f"{path}: bad magic {magic!r}")
    if version != VERSION:
        raise ValueError(f"{path}: unsupported version {version}")
    return b, v


def write_logits(batch, path) -> None:
    """Write a LogitBatch (or a [B, V] numpy array / torch tensor, any device, fp32 or bf16)."""
    values = batch.values if isinstance(batch, LogitBatch) else batch
    if _is_tensor(values):
        values = values.detach().to(torch.float32).cpu().numpy()
    values = np.ascontiguousarray(values, dtype="<f4")
    if values.ndim != 2:
        raise ValueError("logit batch must be 2-D (rows x vocab)")
    with open(path, "wb") as fh:
        fh.write(_HEADER.pack(MAGIC, VERSION, values.shape[0], values.shape[1]))
        fh.write(values.tobytes())


def read_logits(path, device=None) -> LogitBatch:
    """Read a QRTL file.  device=None: a numpy float32 batch (the reference's behaviour);
    device="cuda[:i]": the values go straight to that GPU through page-locked staging."""
    with open(path, "rb") as fh:
        b, v = _read_header(fh, path)
        expected = b * v * 4
        size = os.fstat(fh.fileno()).st_size - _HEADER.size
        if size != expected:
            raise ValueError(f"{path}: expected {expected} payload bytes, got {size}")
        if device is None:
            values = np.frombuffer(fh.read(), dtype="<f4").reshape(b, v)
            return LogitBatch(values.copy())
        staging = torch.empty((b, v), dtype=torch.float32, pin_memory=True)
        if fh.readinto(memoryview(staging.numpy()).cast("B")) != expected:
            raise ValueError(f"{path}: short read")
    return LogitBatch(staging.to(device, non_blocking=False))


def write_targets_csv(targets: TruncTargets, path) -> None:
    """`row,k,p` CSV; p written with repr() so it round-trips exactly (logit_io.py:46-51)."""
    k = targets.k.cpu().numpy() if _is_tensor(targets.k) else np.asarray(targets.k)
    p = targets.p.cpu().numpy() if _is_tensor(targets.p) else np.asarray(targets.p)
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(["row", "k", "p"])
        for i in range(k.shape[0]):
            w.writerow([i, int(k[i]), repr(float(p[i]))])


def read_targets_csv(path) -> TruncTargets:
    """Rows must be 0..B-1 in order under a `row,k,p` header (logit_io.py:54-72)."""
    with open(path, newline="") as fh:
        rows = list(csv.reader(fh))
    if not rows or [c.strip() for c in rows[0]] != ["row", "k", "p"]:
        raise ValueError(f"{path}: expected header 'row,k,p'")
    ks, ps = [], []
    for i, rec in enumerate(rows[1:]):
        if len(rec) != 3:
            raise ValueError(f"{path}: line {i + 2}: expected 3 columns")
        if int(rec[0]) != i:
            raise ValueError(f"{path}: line {i + 2}: rows must be consecutive from 0, got {rec[0]}")
        ks.append(int(rec[1]))
        ps.append(float(rec[2]))
    return TruncTargets(np.array(ks, dtype=np.int64), np.array(ps, dtype=np.float64))
