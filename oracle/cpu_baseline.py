"""CPU baselines for bench.py — TEST / MEASUREMENT INFRASTRUCTURE ONLY (never on the product path).

Times the REFERENCE's own CPU implementation of the hot path on the host cores:

* ``run_batch``   — ``sigmatop.run_batch(LogitBatch, TruncTargets, EngineConfig(threads=1))``
  (pkg/src/sigmatop/engine.py:82-113), fanned out over one process per core on contiguous row
  chunks: SURVEY.md §8d CPU baseline 2 (the reference's thread pool is GIL-bound, baseline 1 ≈ one
  core).  Output is byte-identical to a single call (rows are independent, engine.py:82-101).
* ``sort_select`` — ``sigmatop.engine.sort_select`` (engine.py:183-205), the sort-based definition
  (SURVEY.md §8d baseline 3, Table 3 run J).

The reference is imported from ``baseline/_ref`` (its unmodified pip install; it travels to the GPU
box with the repo).  When it is absent the oracle restatement (oracle/qrita_oracle.py) is timed
instead and the result says ``kind: "port"``.

The pool is created once, outside any timed region: the batch lives in shared memory (written once
by the parent), every worker imports the reference at start-up, and a timed step only sends row
ranges and waits.  Workers write their masked rows into a shared output matrix.
"""
from __future__ import annotations

import concurrent.futures as cf
import multiprocessing as mp
import os
import sys
import time
from multiprocessing import shared_memory

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DIR = os.path.join(ROOT, "baseline", "_ref")

_W = {}


def reference_available() -> tuple:
    """(True, version) if the reference package imports from baseline/_ref, else (False, why)."""
    if not os.path.isdir(os.path.join(REF_DIR, "sigmatop")):
        return False, f"{REF_DIR} has no sigmatop install"
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import sigmatop  # noqa: F401
        return True, getattr(sigmatop, "__version__", "?")
    except Exception as exc:  # pragma: no cover - reported, not raised
        return False, f"import failed: {exc!r}"


def _init(names, shape, k, p, kind):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    shm_in = shared_memory.SharedMemory(name=names[0])
    shm_out = shared_memory.SharedMemory(name=names[1])
    _W["shm"] = (shm_in, shm_out)
    _W["x"] = np.ndarray(shape, dtype=np.float32, buffer=shm_in.buf)
    _W["out"] = np.ndarray(shape, dtype=np.float32, buffer=shm_out.buf)
    _W["k"], _W["p"], _W["kind"] = k, p, kind
    if kind in ("run_batch", "sort_select"):
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        import sigmatop  # noqa: F401
        import sigmatop.engine  # noqa: F401
    else:
        if ROOT not in sys.path:
            sys.path.insert(0, ROOT)
        import oracle.qrita_oracle  # noqa: F401


def _rows(lo: int, hi: int) -> int:
    x, k, p, kind = _W["x"], _W["k"], _W["p"], _W["kind"]
    if kind == "run_batch":
        import sigmatop
        out, _ = sigmatop.run_batch(sigmatop.LogitBatch(x[lo:hi]), sigmatop.TruncTargets(k[lo:hi], p[lo:hi]),
                                    sigmatop.EngineConfig(threads=1))
        _W["out"][lo:hi] = out
    elif kind == "sort_select":
        import sigmatop
        from sigmatop.engine import sort_select
        _W["out"][lo:hi] = sort_select(sigmatop.LogitBatch(x[lo:hi]), sigmatop.TruncTargets(k[lo:hi], p[lo:hi]))
    else:
        from oracle.qrita_oracle import oracle_batch
        out, _ = oracle_batch(x[lo:hi], k[lo:hi], p[lo:hi])
        _W["out"][lo:hi] = out
    return hi - lo


def _noop(_):
    return os.getpid()


class CpuPool:
    """Persistent pool of `procs` worker processes over one shared [B, V] fp32 batch."""

    def __init__(self, x: np.ndarray, k: np.ndarray, p: np.ndarray, procs: int, kind: str = "run_batch"):
        if kind not in ("run_batch", "sort_select", "port"):
            raise ValueError(kind)
        x = np.ascontiguousarray(x, dtype=np.float32)
        self.shape, self.kind, self.procs = x.shape, kind, procs
        self.shm_in = shared_memory.SharedMemory(create=True, size=max(1, x.nbytes))
        self.shm_out = shared_memory.SharedMemory(create=True, size=max(1, x.nbytes))
        np.ndarray(x.shape, dtype=np.float32, buffer=self.shm_in.buf)[...] = x
        self.out = np.ndarray(x.shape, dtype=np.float32, buffer=self.shm_out.buf)
        t0 = time.perf_counter()
        self.ex = cf.ProcessPoolExecutor(max_workers=procs, mp_context=mp.get_context("spawn"),
                                         initializer=_init,
                                         initargs=((self.shm_in.name, self.shm_out.name), x.shape,
                                                   np.asarray(k, np.int64), np.asarray(p, np.float64), kind))
        # start every worker (spawn + reference import) before anything is timed
        list(self.ex.map(_noop, range(4 * procs)))
        self.startup_s = time.perf_counter() - t0

    def run(self, rows: np.ndarray) -> float:
        """Truncate the given rows (sorted, contiguous ranges split over the workers); returns the
        wall seconds of this step."""
        rows = np.asarray(rows)
        lo, hi = int(rows[0]), int(rows[-1]) + 1
        assert hi - lo == rows.size, "rows must be one contiguous range"
        n = hi - lo
        parts = [(lo + n * i // self.procs, lo + n * (i + 1) // self.procs) for i in range(self.procs)]
        t0 = time.perf_counter()
        futs = [self.ex.submit(_rows, a, b) for a, b in parts if b > a]
        done = sum(f.result() for f in futs)
        wall = time.perf_counter() - t0
        assert done == n
        return wall

    def close(self):
        self.ex.shutdown(wait=True)
        self.out = None  # drop the view before the segment is closed
        for s in (self.shm_in, self.shm_out):
            s.close()
            s.unlink()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
