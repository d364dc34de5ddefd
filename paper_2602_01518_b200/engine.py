"""Batch driver — the drop-in for the reference's engine.py (pkg/src/sigmatop/engine.py:26-237).

`run_batch` is the boundary the reference's callers use (engine.py:82-113): same arguments, same
(outputs, BatchReport) result, same ValueError on invalid input.  Rows are processed by one launch of
the B200 kernels instead of a GIL-bound thread pool; `EngineConfig.threads` is accepted and
validated for compatibility (output never depended on it, test_acceptance.py:177-199).
"""
from __future__ import annotations

import csv
import ctypes
import statistics
import time
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np
import torch

from . import _native as N
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
        x = torch.from_numpy(np.ascontiguousarray(x)).to(dev)
    elif not x.is_cuda:
        x = x.to(dev)
    k = targets.k if _is_tensor(targets.k) else torch.from_numpy(np.ascontiguousarray(targets.k))
    p = targets.p if _is_tensor(targets.p) else torch.from_numpy(np.ascontiguousarray(targets.p))
    return x, k.to(dev, torch.int64), p.to(dev, torch.float64)


_METRICS_DTYPE = np.dtype([("trunc_hit", "<i4"), ("outlier_count", "<i4"), ("outlier_prob_sum", "<f8"),
                           ("k_search_iters", "<i4"), ("p_search_iters", "<i4"), ("fallback_used", "<i4"),
                           ("kept_count", "<i4"), ("full_row_path", "<i4"), ("row_passes", "<i4")])
assert _METRICS_DTYPE.itemsize == 40  # qrita_row_metrics (include/qrita_b200.h)


def metrics_to_rows(buf: torch.Tensor) -> List[RowMetrics]:
    m = np.frombuffer(buf.cpu().numpy().tobytes(), dtype=_METRICS_DTYPE)
    return [RowMetrics(trunc_hit=bool(h), outlier_count=int(c), outlier_prob_sum=float(s),
                       k_search_iters=int(ik), p_search_iters=int(ip), fallback_used=bool(f))
            for h, c, s, ik, ip, f in zip(m["trunc_hit"].tolist(), m["outlier_count"].tolist(),
                                          m["outlier_prob_sum"].tolist(), m["k_search_iters"].tolist(),
                                          m["p_search_iters"].tolist(), m["fallback_used"].tolist())]


def _host_targets_ok(batch: LogitBatch, targets: TruncTargets) -> bool:
    """The O(B) part of validate_batch (lengths, k in [1, V], p in (0, 1]), vectorised; the O(B*V)
    finiteness check runs on the device, fused into the truncation kernel (status block)."""
    k = targets.k.cpu().numpy() if _is_tensor(targets.k) else np.asarray(targets.k)
    p = targets.p.cpu().numpy() if _is_tensor(targets.p) else np.asarray(targets.p)
    b, v = batch.batch_size, batch.vocab_size
    return (k.shape == (b,) and p.shape == (b,) and bool(np.all((k >= 1) & (k <= v)))
            and bool(np.all((p > 0.0) & (p <= 1.0))))


def run_batch(batch: LogitBatch, targets: TruncTargets, config: EngineConfig, *, devices=None):
    """Truncate every row (engine.py:82-113).  Returns (outputs, BatchReport).

    numpy input -> numpy float32 output (the reference's contract), through the library's native
    host-buffer pipeline (qrita_topk_topp_host: row chunks copied in, truncated and copied back with
    both PCIe directions overlapped with the kernels); CUDA tensor input -> CUDA tensor output in the
    input dtype, one stream-ordered launch.  Invalid input raises the reference's
    ValueError("invalid batch: ...") with the reference's report lines; logit finiteness is checked
    on the device (fused into the kernel), k / p on the host.  devices=[...] shards the rows over
    several GPUs in contiguous blocks (sharded.topk_topp_sharded).
    """
    if not isinstance(batch, LogitBatch):
        batch = LogitBatch(batch)
    if not _host_targets_ok(batch, targets):
        _check_inputs(batch, targets)      # the reference's full report (raises)
    b = batch.batch_size
    on_gpu = _is_tensor(batch.values) and batch.values.is_cuda
    if devices is not None and len(devices) > 1:
        dev = torch.device("cuda", torch.cuda.current_device()) if not on_gpu else batch.values.device
    elif devices is not None:
        dev = torch.device(devices[0]) if not isinstance(devices[0], int) else torch.device("cuda", devices[0])
    else:
        dev = batch.values.device if on_gpu else torch.device("cuda", torch.cuda.current_device())
    try:
        if on_gpu:
            x, k, p = _device_inputs(batch, targets, dev)
            met = ops.metrics_buffer(b, x.device)
            torch.cuda.synchronize(x.device)
            start = time.perf_counter_ns()
            if devices is not None and len(devices) > 1:
                out = _sharded(x, k, p, config, devices, met)
            else:
                out = ops.topk_topp(x, k, p, flags=config.flags(), sample_size=config.sample_size,
                                    metrics=met, check=True)
            torch.cuda.synchronize(x.device)
            wall = time.perf_counter_ns() - start
        else:
            vals = batch.values
            xh = vals if _is_tensor(vals) else torch.from_numpy(np.ascontiguousarray(vals))
            kh = targets.k.cpu() if _is_tensor(targets.k) else torch.from_numpy(np.asarray(targets.k, np.int64))
            ph = targets.p.cpu() if _is_tensor(targets.p) else torch.from_numpy(np.asarray(targets.p, np.float64))
            # the numpy result lives in page-locked memory from torch's caching host allocator (the array
            # keeps the block alive): downloads go straight into it, and no fresh pages are faulted in
            oh = torch.empty((b, batch.vocab_size), dtype=torch.float32, pin_memory=True) \
                if not _is_tensor(vals) else torch.empty_like(xh, pin_memory=True)
            res = oh.numpy() if not _is_tensor(vals) else None
            met = ops.metrics_buffer(b, dev)
            start = time.perf_counter_ns()
            if devices is not None and len(devices) > 1:
                out = _sharded(xh, kh, ph, config, devices, met, out=oh)
            else:
                out = ops.topk_topp_host(xh, kh, ph, out=oh, flags=config.flags(), sample_size=config.sample_size,
                                         metrics=met, check=True, device=dev)
            wall = time.perf_counter_ns() - start
            out = res if res is not None else out
    except ops.TruncationError:
        _check_inputs(batch, targets)      # the reference's exact report lines (raises)
        raise
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
    return out, report


def _sharded(x, k, p, config: EngineConfig, devices, met: torch.Tensor, out=None):
    """run_batch over several devices: per-block metrics are gathered into `met` (on its device)."""
    from .sharded import topk_topp_sharded
    res = topk_topp_sharded(x, k, p, devices, out=out, flags=config.flags(), sample_size=config.sample_size,
                            check=True, metrics=met)
    return res


def verify_batch(batch: LogitBatch, targets: TruncTargets, config: EngineConfig,
                 reference: Optional[Callable] = None) -> List[Divergence]:
    """Differential check (engine.py:116-136): this build against a reference row function
    `reference(row, k, p) -> masked_row` (numpy).  Default reference: the exact sort-based GPU
    selection `sort_select` (an independent code path: stable sort + exact prefix masses), under the
    config's duplicate-handling semantics."""
    _check_inputs(batch, targets)
    got, _ = run_batch(batch, targets, config)
    got = got if not _is_tensor(got) else got.float().cpu().numpy()
    if reference is None:
        want = sort_select(batch, targets, dup_handling=config.duplication_handling_enabled)
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
                sample_size: int = ops.DEFAULT_SAMPLE_SIZE, dup_handling: bool = True):
    """Sort-based selection (engine.py:183-205), exact, on the GPU: stable descending sort, top-k
    prefix, fp64 softmax over the survivors, exact prefix masses (sortsel.py).  Independent of the
    pivot-search kernels; verify_batch's default reference and Table 3 runs I / J.

    use_sigma_trunc=True (run I): rows with k != V whose sigma pre-filter hits (count > k,
    sigma_trunc.py:127-138) sort only their outliers — the entries above t = mu + delta_adj * sigma,
    in index order — exactly as the reference does (engine.py:190-201); the answer is the same.
    dup_handling=False: the pipeline's whole-cluster rule (Table 3 runs C / E) instead of the
    oracle's."""
    from . import sigma as S
    from .sortsel import exact_sort_topk_topp
    _check_inputs(batch, targets)
    x, k, p = _device_inputs(batch, targets)
    b, v = x.shape
    out = None
    if use_sigma_trunc:
        kk = k.cpu().numpy()
        rows = [i for i in range(b) if kk[i] != v]
        if rows:
            xs = x[rows].contiguous()
            stats = torch.empty((len(rows), 2), dtype=torch.float64, device=x.device)
            st = torch.cuda.current_stream(x.device)
            rc = N.load().qrita_row_stats(ctypes.c_void_p(xs.data_ptr()), v, ops._DTYPES[xs.dtype], len(rows), v,
                                          int(sample_size), ctypes.c_void_p(stats.data_ptr()),
                                          ctypes.c_void_p(st.cuda_stream))
            if rc != N.OK:
                raise RuntimeError(f"qrita_row_stats failed: {N.strerror(rc)}")
            mu_sig = stats.cpu().numpy()
            out = torch.empty_like(x)
            done = np.zeros(b, dtype=bool)
            for j, i in enumerate(rows):
                delta = S.lookup_delta_topk(int(kk[i]), v)
                t = S.threshold_from(S.GaussianStats(float(mu_sig[j, 0]), float(mu_sig[j, 1]), sample_size), delta).t
                z = x[i].to(torch.float64)
                idx = torch.nonzero(z > t, as_tuple=True)[0]
                if idx.numel() > int(kk[i]):                 # hit: sort the outliers only
                    sub = exact_sort_topk_topp(x[i, idx].unsqueeze(0), k[i:i + 1], p[i:i + 1],
                                               dup_handling=dup_handling)[0]
                    out[i].fill_(float("-inf"))
                    out[i, idx] = sub
                    done[i] = True
            rest = np.nonzero(~done)[0]
            if rest.size:
                ri = torch.as_tensor(rest, device=x.device)
                out[ri] = exact_sort_topk_topp(x[ri], k[ri], p[ri], dup_handling=dup_handling)
    if out is None:
        out = exact_sort_topk_topp(x, k, p, dup_handling=dup_handling)
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


def report_row(run_id: str, batch: LogitBatch, targets: TruncTargets, config: EngineConfig,
               report: BatchReport) -> dict:
    """One aggregate CSV row in the fixed report schema (engine.py:240-262).  The search-iteration
    means are this build's integer-key pivot passes (RowMetrics note in core.py)."""
    kk = targets.k.cpu().numpy() if _is_tensor(targets.k) else np.asarray(targets.k)
    pp = targets.p.cpu().numpy() if _is_tensor(targets.p) else np.asarray(targets.p)
    ks, ps = np.unique(kk), np.unique(pp)
    return {
        "run_id": run_id, "B": batch.batch_size, "V": batch.vocab_size,
        "k": int(ks[0]) if ks.shape[0] == 1 else "rand",
        "p": float(ps[0]) if ps.shape[0] == 1 else "rand",
        "search_kind": config.search_kind,
        "trunc_enabled": config.sigma_trunc_enabled and not config.force_fallback,
        "dup_enabled": config.duplication_handling_enabled,
        "hit_rate": report.hit_rate, "mean_outliers": report.mean_outliers,
        "mean_prob_sum": report.mean_prob_sum, "mean_iters_k": report.mean_iters_k,
        "mean_iters_p": report.mean_iters_p, "wall_ms": report.wall_time_ns / 1e6,
        "rows_per_s": report.rows_per_second,
    }


def write_report_csv(rows: List[dict], path, columns: Optional[List[str]] = None) -> None:
    """CSV in the reference's fixed schema (engine.py:265-269); `columns` may append extra columns
    (the B200 bench adds the parity tag of each run)."""
    cols = columns or REPORT_COLUMNS
    with open(path, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=cols, lineterminator="\n")
        w.writeheader()
        for r in rows:
            w.writerow({c: r.get(c, "") for c in cols})
