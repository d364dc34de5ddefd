"""Batch driver — the drop-in for the reference's engine.py (pkg/src/sigmatop/engine.py:26-237).

`run_batch` is the boundary the reference's callers use (engine.py:82-113): same arguments, same
(outputs, BatchReport) result, same ValueError on invalid input.  Rows are processed by one launch of
the B200 kernels instead of a GIL-bound thread pool; `EngineConfig.threads` is accepted and
validated for compatibility (output never depended on it, test_acceptance.py:177-199).
"""
from __future__ import annotations

import statistics
import time
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np
import torch

from . import ops
from .core import LogitBatch, RowMetrics, Tolerances, TruncTargets, _is_tensor, validate_batch

REPORT_COLUMNS = ["run_id", "B", "V", "k", "p", "search_kind", "trunc_enabled",
                  "dup_enabled", "hit_rate", "mean_outliers", "mean_prob_sum",
                  "mean_iters_k", "mean_iters_p", "wall_ms", "rows_per_s"]


@dataclass(frozen=True)
class EngineConfig:
    """engine.py:26-40."""

    threads: int = 1
    search_kind: str = "quaternary"
    sigma_trunc_enabled: bool = True
    duplication_handling_enabled: bool = True
    force_fallback: bool = False
    sample_size: int = ops.DEFAULT_SAMPLE_SIZE
    tolerances: Tolerances = field(default_factory=Tolerances)

    def __post_init__(self):
        if self.threads < 1:
            raise ValueError("threads must be >= 1")
        if self.search_kind not in ("quaternary", "binary"):
            raise ValueError("search_kind must be 'quaternary' or 'binary'")

    def flags(self) -> ops.TruncFlags:
        return ops.TruncFlags(search=self.search_kind, use_sigma_trunc=self.sigma_trunc_enabled,
                              force_fallback=self.force_fallback,
                              dup_handling=self.duplication_handling_enabled)


@dataclass
class BatchReport:
    """engine.py:43-52."""

    per_row: List[RowMetrics]
    hit_rate: float
    mean_outliers: float
    mean_prob_sum: float
    mean_iters_k: float
    mean_iters_p: float
    wall_time_ns: int
    rows_per_second: float


@dataclass
class Divergence:
    """First mismatching entry of a row plus the mismatch count (engine.py:55-63)."""

    row: int
    index: int
    got: float
    expected: float
    n_mismatch: int


def _check_inputs(batch: LogitBatch, targets: TruncTargets):
    report = validate_batch(batch, targets)
    if report:
        raise ValueError("invalid batch: " + "; ".join(report[:5]))


def _device_inputs(batch: LogitBatch, targets: TruncTargets, device=None):
    dev = torch.device(device) if device is not None else (
        batch.values.device if _is_tensor(batch.values) and batch.values.is_cuda
        else torch.device("cuda", torch.cuda.current_device()))
    x = batch.values
    if not _is_tensor(x):
        x = torch.from_numpy(np.ascontiguousarray(x)).pin_memory().to(dev, non_blocking=True)
    elif not x.is_cuda:
        x = x.to(dev)
    k = targets.k if _is_tensor(targets.k) else torch.from_numpy(np.ascontiguousarray(targets.k))
    p = targets.p if _is_tensor(targets.p) else torch.from_numpy(np.ascontiguousarray(targets.p))
    return x, k.to(dev, torch.int64), p.to(dev, torch.float64)


def metrics_to_rows(buf: torch.Tensor) -> List[RowMetrics]:
    rows = []
    for m in ops.decode_metrics(buf):
        rows.append(RowMetrics(trunc_hit=bool(m["trunc_hit"]), outlier_count=int(m["outlier_count"]),
                               outlier_prob_sum=float(m["outlier_prob_sum"]),
                               k_search_iters=int(m["k_search_iters"]),
                               p_search_iters=int(m["p_search_iters"]),
                               fallback_used=bool(m["fallback_used"])))
    return rows


def run_batch(batch: LogitBatch, targets: TruncTargets, config: EngineConfig):
    """Truncate every row (engine.py:82-113).  Returns (outputs, BatchReport).

    numpy input -> numpy float32 output (the reference's contract); CUDA tensor input -> CUDA
    tensor output in the input dtype.
    """
    if not isinstance(batch, LogitBatch):
        batch = LogitBatch(batch)
    _check_inputs(batch, targets)
    x, k, p = _device_inputs(batch, targets)
    b = batch.batch_size
    met = ops.metrics_buffer(b, x.device)
    torch.cuda.synchronize(x.device)
    start = time.perf_counter_ns()
    out = ops.topk_topp(x, k, p, flags=config.flags(), sample_size=config.sample_size,
                        metrics=met, check=False)
    torch.cuda.synchronize(x.device)
    wall = time.perf_counter_ns() - start
    per_row = metrics_to_rows(met)
    report = BatchReport(
        per_row=per_row,
        hit_rate=sum(m.trunc_hit for m in per_row) / b,
        mean_outliers=sum(m.outlier_count for m in per_row) / b,
        mean_prob_sum=sum(m.outlier_prob_sum for m in per_row) / b,
        mean_iters_k=sum(m.k_search_iters for m in per_row) / b,
        mean_iters_p=sum(m.p_search_iters for m in per_row) / b,
        wall_time_ns=wall,
        rows_per_second=b / (wall / 1e9) if wall > 0 else float("inf"))
    if not _is_tensor(batch.values):
        out = out.cpu().numpy()
    return out, report


def verify_batch(batch: LogitBatch, targets: TruncTargets, config: EngineConfig,
                 reference: Optional[Callable] = None) -> List[Divergence]:
    """Differential check (engine.py:116-136): this build against a reference row function
    `reference(row, k, p) -> masked_row` (numpy).  Default reference: the exact sort-based GPU
    selection `sort_select` (an independent code path: stable sort + exact prefix masses)."""
    _check_inputs(batch, targets)
    got, _ = run_batch(batch, targets, config)
    got = got if not _is_tensor(got) else got.float().cpu().numpy()
    if reference is None:
        want = sort_select(batch, targets)
        want = want if not _is_tensor(want) else want.float().cpu().numpy()
    else:
        xs = batch.values if not _is_tensor(batch.values) else batch.values.float().cpu().numpy()
        kk = np.asarray(targets.k if not _is_tensor(targets.k) else targets.k.cpu())
        pp = np.asarray(targets.p if not _is_tensor(targets.p) else targets.p.cpu())
        want = np.stack([np.asarray(reference(xs[i], int(kk[i]), float(pp[i])))
                         for i in range(batch.batch_size)])
    divs = []
    for i in range(batch.batch_size):
        g, w = got[i], want[i]
        same = (g.view(np.uint32) == w.view(np.uint32)) | (np.isneginf(g) & np.isneginf(w))
        if not same.all():
            bad = np.nonzero(~same)[0]
            j = int(bad[0])
            divs.append(Divergence(row=i, index=j, got=float(g[j]), expected=float(w[j]),
                                   n_mismatch=int(bad.shape[0])))
    return divs


def synth_batch(kind: str, batch_size: int, vocab_size: int, seed: int, **params) -> LogitBatch:
    """Seeded synthetic batches (engine.py:139-180): gaussian, gaussian_outliers, quantized,
    uniform.  The same seed draws the same float32 matrix as the reference."""
    if batch_size < 1 or vocab_size < 1:
        raise ValueError("batch_size and vocab_size must be >= 1")
    rng = np.random.default_rng(seed)
    if kind == "gaussian":
        vals = rng.normal(params.pop("mu0", 0.0), params.pop("sigma0", 1.0),
                          size=(batch_size, vocab_size))
    elif kind == "gaussian_outliers":
        m = int(params.pop("m", 50))
        magnitude = params.pop("magnitude", 12.0)
        if not 0 <= m <= vocab_size:
            raise ValueError("m must be in [0, V]")
        vals = rng.normal(0.0, 1.0, size=(batch_size, vocab_size))
        for r in range(batch_size):
            cols = rng.choice(vocab_size, size=m, replace=False)
            vals[r, cols] = magnitude + rng.random(m)
    elif kind == "quantized":
        g = int(params.pop("g", 16))
        if g < 1:
            raise ValueError("g must be >= 1")
        levels = np.linspace(-3.0, 3.0, g)
        z = np.clip(rng.normal(0.0, 1.0, size=(batch_size, vocab_size)), -3, 3)
        if vocab_size * batch_size <= 1 << 20:
            vals = levels[np.argmin(np.abs(z[..., None] - levels), axis=-1)]
        else:
            vals = levels[np.clip(np.round((z + 3.0) / 6.0 * (g - 1)).astype(np.int64), 0, g - 1)]
    elif kind == "uniform":
        vals = rng.uniform(params.pop("low", 0.0), params.pop("high", 1.0),
                           size=(batch_size, vocab_size))
    else:
        raise ValueError(f"unknown batch kind {kind!r}")
    if params:
        raise ValueError(f"unused params for kind {kind!r}: {sorted(params)}")
    return LogitBatch(vals.astype(np.float32))


def sort_select(batch: LogitBatch, targets: TruncTargets, use_sigma_trunc: bool = False,
                sample_size: int = ops.DEFAULT_SAMPLE_SIZE):
    """Sort-based selection (engine.py:183-205), exact, on the GPU: stable descending sort, top-k
    prefix, fp64 softmax over the survivors, exact prefix masses (sortsel.py).  Independent of the
    pivot-search kernels; used as verify_batch's default reference and as a bench baseline."""
    from .sortsel import exact_sort_topk_topp
    _check_inputs(batch, targets)
    x, k, p = _device_inputs(batch, targets)
    out = exact_sort_topk_topp(x, k, p)
    return out if _is_tensor(batch.values) else out.cpu().numpy()


def bench(batch: LogitBatch, targets: TruncTargets, config: EngineConfig, repeats: int = 5):
    """Median / min wall time of this build and of the sort baseline (engine.py:208-237)."""
    if repeats < 3:
        raise ValueError("repeats must be >= 3")
    _check_inputs(batch, targets)
    x, k, p = _device_inputs(batch, targets)
    flags = config.flags()

    def time_fn(fn):
        fn()
        torch.cuda.synchronize()
        times = []
        for _ in range(repeats):
            t0 = time.perf_counter_ns()
            fn()
            torch.cuda.synchronize()
            times.append(time.perf_counter_ns() - t0)
        return times

    from .sortsel import exact_sort_topk_topp
    pipe = time_fn(lambda: ops.topk_topp(x, k, p, flags=flags, sample_size=config.sample_size,
                                         check=False))
    oracle = time_fn(lambda: exact_sort_topk_topp(x, k, p))

    def row(name, times):
        med = statistics.median(times)
        return {"method": name, "median_ms": med / 1e6, "min_ms": min(times) / 1e6,
                "rows_per_s": batch.batch_size / (med / 1e9)}

    return [row("pipeline", pipe), row("sort_oracle", oracle)]
