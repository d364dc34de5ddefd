"""The reference's sigma_trunc surface (pkg/src/sigmatop/sigma_trunc.py) for drop-in callers.

The fused kernel runs this pre-filter internally (csrc/qrita_plan.cuh); these are the standalone
primitives with the reference's names, dataclasses, argument checks and arithmetic:

* ``TOPK_TABLE`` / ``TOPP_TABLE`` — the embedded 200-entry quantile tables, read from the library
  (``qrita_sigma_table``: one copy of the numbers for the kernels and for Python);
* ``row_stats`` — on the GPU (``qrita_row_stats``): numpy's pairwise mean / mean square of the first
  ``min(sample_size, V)`` entries bit for bit (sigma_trunc.py:69-82);
* ``lookup_delta_topk`` / ``lookup_delta_topp`` / ``threshold_from`` / ``is_hit`` — scalar
  arithmetic, same expressions (sigma_trunc.py:85-103, 127-138);
* ``gather_outliers`` — stable compaction of ``z > t`` on the GPU (sigma_trunc.py:106-124);
* ``generate_table_entries`` / ``generate_table`` — Monte-Carlo table regeneration
  (sigma_trunc.py:141-185): the reference's N(0,1) draw (numpy's generator, so a seed gives the same
  sample), sorted and integrated on the GPU; ``profile_tables`` derives tables from real logits.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _native as N
from . import ops
from .core import _is_tensor, stable_softmax

TABLE_SIZE = 200               # tables.py:11
SAFETY_MARGIN = 0.2            # sigma_trunc.py:20
DEFAULT_SAMPLE_SIZE = ops.DEFAULT_SAMPLE_SIZE


@dataclass(frozen=True)
class GaussianStats:
    mu: float
    sigma: float
    sample_size: int


@dataclass(frozen=True)
class SigmaTable:
    """200-entry quantile table; kind is 'topk' or 'topp' (sigma_trunc.py:31-48)."""

    entries: np.ndarray
    kind: str

    def __post_init__(self):
        e = np.asarray(self.entries, dtype=np.float64)
        if e.shape != (TABLE_SIZE,):
            raise ValueError(f"table must have exactly {TABLE_SIZE} entries")
        if self.kind not in ("topk", "topp"):
            raise ValueError("kind must be 'topk' or 'topp'")
        object.__setattr__(self, "entries", e)


@dataclass(frozen=True)
class TruncThreshold:
    delta_raw: float
    delta_adj: float
    t: float


@dataclass(frozen=True)
class OutlierSet:
    """Stable compaction of all row entries strictly above the threshold."""

    values: object
    count: int
    row_max: float
    row_min: float
    prob_sum: Optional[float] = None


def _library_table(kind: int) -> np.ndarray:
    out = np.empty(TABLE_SIZE, dtype=np.float64)
    if N.load().qrita_sigma_table(kind, out.ctypes.data, TABLE_SIZE) != N.OK:
        raise RuntimeError("qrita_sigma_table failed")
    return out


_TABLES = {}


def __getattr__(name):
    # TOPK_TABLE / TOPP_TABLE are read from the library on first use, so importing the package does
    # not need the built library (the build step imports it)
    if name in ("TOPK_TABLE", "TOPP_TABLE"):
        if name not in _TABLES:
            _TABLES[name] = SigmaTable(_library_table(0 if name == "TOPK_TABLE" else 1),
                                       "topk" if name == "TOPK_TABLE" else "topp")
        return _TABLES[name]
    raise AttributeError(name)


def _row_tensor(row) -> torch.Tensor:
    if _is_tensor(row):
        t = row if row.is_cuda else row.to("cuda")
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(row, dtype=np.float32))).to("cuda")
    if t.dtype not in ops._DTYPES:
        t = t.to(torch.float32)
    return t


def row_stats(row, sample_size: int = DEFAULT_SAMPLE_SIZE) -> GaussianStats:
    """Mean / std of the first min(sample_size, V) entries at 64-bit, variance floored at zero
    (sigma_trunc.py:69-82), computed on the GPU with numpy's pairwise summation order."""
    if sample_size < 1:
        raise ValueError("sample_size must be >= 1")
    t = _row_tensor(row).reshape(1, -1).contiguous()
    v = t.shape[1]
    out = torch.empty(2, dtype=torch.float64, device=t.device)
    st = torch.cuda.current_stream(t.device)
    rc = N.load().qrita_row_stats(ctypes.c_void_p(t.data_ptr()), v, ops._DTYPES[t.dtype], 1, v, int(sample_size),
                                  ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(st.cuda_stream))
    if rc != N.OK:
        raise RuntimeError(f"qrita_row_stats failed: {N.strerror(rc)}")
    mu, sigma = out.tolist()
    return GaussianStats(mu=mu, sigma=sigma, sample_size=min(sample_size, v))


def lookup_delta_topk(k: int, vocab_size: int, table: Optional[SigmaTable] = None) -> float:
    table = table or __getattr__("TOPK_TABLE")
    if not 1 <= k <= vocab_size:
        raise ValueError("k must be in [1, V]")
    idx = min(int(k / vocab_size * TABLE_SIZE), TABLE_SIZE - 1)
    return float(table.entries[idx])


def lookup_delta_topp(p: float, table: Optional[SigmaTable] = None) -> float:
    table = table or __getattr__("TOPP_TABLE")
    if not 0.0 < p <= 1.0:
        raise ValueError("p must be in (0, 1]")
    idx = min(int(p * TABLE_SIZE), TABLE_SIZE - 1)
    return float(table.entries[idx])


def threshold_from(stats: GaussianStats, delta: float) -> TruncThreshold:
    """Safety margin on delta, then t = mu + delta_adj * sigma (sigma_trunc.py:99-103)."""
    delta_adj = delta - SAFETY_MARGIN * abs(delta)
    return TruncThreshold(delta_raw=delta, delta_adj=delta_adj, t=stats.mu + delta_adj * stats.sigma)


def gather_outliers(row, stats: GaussianStats, delta: float, mode: str = "topk", probs=None) -> OutlierSet:
    """Order-stable compaction of the entries strictly above t, with the row extrema; 'topp' mode also
    sums the outliers' softmax mass (sigma_trunc.py:106-124).  On the GPU; values come back as numpy
    for numpy rows, as a CUDA float64 tensor for tensor rows."""
    thr = threshold_from(stats, delta)
    z = _row_tensor(row).to(torch.float64)
    mask = z > thr.t
    values = z[mask]                       # boolean indexing keeps index order
    prob_sum = None
    if mode == "topp":
        if probs is None:
            probs, _, _ = stable_softmax(row)
        pr = probs if _is_tensor(probs) else torch.as_tensor(np.asarray(probs), device=z.device)
        prob_sum = float(pr.to(z.device)[mask].sum())
    vals = values if _is_tensor(row) else values.cpu().numpy()
    return OutlierSet(values=vals, count=int(values.shape[0]), row_max=float(z.max()), row_min=float(z.min()),
                      prob_sum=prob_sum)


def is_hit(outliers: OutlierSet, k: Optional[int] = None, p: Optional[float] = None, mode: str = "topk") -> bool:
    """top-k: count > k (strict); top-p: outlier mass > p (sigma_trunc.py:127-138)."""
    if mode == "topk":
        return outliers.count > k
    if outliers.prob_sum is None:
        raise ValueError("top-p hit test requires prob_sum")
    return outliers.prob_sum > p


def _host_sample(num_samples: int, seed: int) -> np.ndarray:
    return np.random.default_rng(seed).standard_normal(num_samples)


def _entries_from_sorted(sample_desc: torch.Tensor, kind: str, entries: int) -> np.ndarray:
    n = sample_desc.shape[0]
    dev = sample_desc.device
    if kind == "topk":
        # the ranks are host arithmetic, exactly the reference's expression (sigma_trunc.py:155-157)
        ranks = np.ceil(np.arange(1, entries + 1) / entries * n)
        idx = torch.as_tensor(np.minimum(ranks.astype(np.int64) - 1, n - 1), device=dev)
        return sample_desc[idx].cpu().numpy().copy()
    exps = torch.exp(sample_desc - sample_desc[0])
    probs = exps / exps.sum()
    csum = torch.cumsum(probs, 0)
    targets = torch.as_tensor(np.arange(1, entries + 1) / entries, device=dev)
    idx = torch.clamp(torch.searchsorted(csum, targets, side="left"), max=n - 1)
    return sample_desc[idx].cpu().numpy().copy()


def generate_table_entries(kind: str, num_samples: int, seed: int, entries: int = TABLE_SIZE) -> np.ndarray:
    """Monte-Carlo regeneration of table entries (sigma_trunc.py:141-166): the same N(0,1) sample as
    the reference (numpy's generator and seed), sorted descending and integrated on the GPU.  topk:
    entry i is the sample at descending rank ceil((i+1)/n * N); topp: the sample where the descending
    cumulative softmax mass first reaches (i+1)/n.  (Softmax sums run in fp64 on the GPU, so a topp
    entry can differ from the reference's sequential cumsum where two cumulative masses straddle a
    target within a few ulps.)"""
    if num_samples < 100_000:
        raise ValueError("num_samples must be >= 100000")
    if kind not in ("topk", "topp"):
        raise ValueError("kind must be 'topk' or 'topp'")
    s = torch.from_numpy(_host_sample(num_samples, seed)).to("cuda")
    s, _ = torch.sort(s, descending=True)
    return _entries_from_sorted(s, kind, entries)


def generate_table(kind: str, num_samples: int, seed: int) -> SigmaTable:
    """Regenerate a standard 200-entry SigmaTable (see generate_table_entries)."""
    return SigmaTable(generate_table_entries(kind, num_samples, seed), kind)


def profile_tables(logits, sample_size: int = DEFAULT_SAMPLE_SIZE, entries: int = TABLE_SIZE):
    """Per-model tables from real logits: every row is
    standardised with its own row_stats (mu, sigma of the first sample_size entries, as the
    pre-filter sees them), the standardised rows are pooled, and the table entries are read off the
    pooled sample exactly like generate_table_entries.  Returns (TOPK table, TOPP table) for
    inspection / lookup_delta_* (the kernels use the embedded tables; a table only moves the hit
    rate, never the output)."""
    x = logits if _is_tensor(logits) else torch.from_numpy(np.ascontiguousarray(logits, dtype=np.float32))
    x = x.to("cuda")
    if x.dim() == 1:
        x = x.unsqueeze(0)
    b, v = x.shape
    xs = x if x.dtype in ops._DTYPES else x.float()
    xs = xs.contiguous()
    stats = torch.empty((b, 2), dtype=torch.float64, device=x.device)
    st = torch.cuda.current_stream(x.device)
    rc = N.load().qrita_row_stats(ctypes.c_void_p(xs.data_ptr()), v, ops._DTYPES[xs.dtype], b, v, int(sample_size),
                                  ctypes.c_void_p(stats.data_ptr()), ctypes.c_void_p(st.cuda_stream))
    if rc != N.OK:
        raise RuntimeError(f"qrita_row_stats failed: {N.strerror(rc)}")
    sig = torch.where(stats[:, 1:] > 0, stats[:, 1:], torch.ones_like(stats[:, 1:]))
    zs = ((x.to(torch.float64) - stats[:, :1]) / sig).reshape(-1)
    zs, _ = torch.sort(zs, descending=True)
    k_entries, p_entries = _entries_from_sorted(zs, "topk", entries), _entries_from_sorted(zs, "topp", entries)
    if entries != TABLE_SIZE:
        return k_entries, p_entries
    return SigmaTable(k_entries, "topk"), SigmaTable(p_entries, "topp")


def write_table_csv(entries, path) -> None:
    """Two-column CSV (index, value), 6-decimal fixed notation (sigma_trunc.py:169-176)."""
    import csv
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(["index", "value"])
        for i, v in enumerate(np.asarray(entries)):
            w.writerow([i, f"{v:.6f}"])


def read_table_csv(path) -> np.ndarray:
    import csv
    with open(path, newline="") as fh:
        rows = list(csv.reader(fh))
    return np.array([float(r[1]) for r in rows[1:]], dtype=np.float64)


__all__ = ["TABLE_SIZE", "SAFETY_MARGIN", "GaussianStats", "SigmaTable", "TruncThreshold", "OutlierSet",
           "TOPK_TABLE", "TOPP_TABLE", "row_stats", "lookup_delta_topk", "lookup_delta_topp", "threshold_from",
           "gather_outliers", "is_hit", "generate_table_entries", "generate_table", "profile_tables",
           "write_table_csv", "read_table_csv"]
