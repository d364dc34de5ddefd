"""Generate the golden fixtures under tests/golden/ from the REFERENCE implementation itself.

Run where the reference tree is mounted (it does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every expected kept set below comes from `sigmatop.oracle.oracle_topk_topp` (the reference's ground
truth, pkg/src/sigmatop/oracle.py:70-89) and every metric from `sigmatop.engine.run_batch`
(engine.py:82-113).  Inputs are regenerated from seeds at test time by oracle/synth.py; their sha256
is stored so a drifting RNG is caught instead of silently changing the expected answers.

Kept sets are stored exactly but compactly as (boundary value bits, cut index, kept count):
kept(i) <=> z_i > z_b or (z_i == z_b and i <= cut) — this is verified against the full mask for
every stored row before it is written.
"""
from __future__ import annotations

import itertools
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import sigmatop  # noqa: E402  (the reference package)
from sigmatop.core import LogitBatch, TruncTargets  # noqa: E402
from sigmatop.engine import EngineConfig, run_batch  # noqa: E402
from sigmatop.oracle import oracle_topk_topp  # noqa: E402

from oracle.qrita_oracle import boundary_of_mask, mask_from_boundary  # noqa: E402
from oracle.synth import config_inputs, sha256, synth  # noqa: E402


def ref_keep(row, k, p):
    out = oracle_topk_topp(np.asarray(row, dtype=np.float32), int(k), float(p)).masked_row
    return ~np.isneginf(out)


def triplet(row, keep):
    zb, cut, cnt = boundary_of_mask(row, keep)
    assert np.array_equal(mask_from_boundary(row, zb, cut), keep), "boundary encoding not exact"
    return zb, cut, cnt


def ref_metrics(x, k, p):
    _, rep = run_batch(LogitBatch(x), TruncTargets(k, p), EngineConfig())
    m = rep.per_row
    return {
        "trunc_hit": np.array([r.trunc_hit for r in m], dtype=np.int8),
        "outlier_count": np.array([r.outlier_count for r in m], dtype=np.int64),
        "outlier_prob_sum": np.array([r.outlier_prob_sum for r in m], dtype=np.float64),
        "fallback_used": np.array([r.fallback_used for r in m], dtype=np.int8),
    }


def kats():
    """Known answers of the reference's own unit tests (test_oracle.py:10-44, test_pipeline.py)."""
    cases = [
        ([3, 2, 1, 0], 2, 1.0), ([1, 1, 1, 1], 2, 1.0), ([5, 5, 3, 5, 1], 2, 1.0),
        ([2, 1, 0], 3, 0.7), ([7, 7, 7], 3, 1.0), ([0, 0, 0, 0], 4, 0.5),
        ([2, 1, 0, -1], 3, 0.9), ([2, 2, 2, 1], 2, 1.0), ([1, 2, 2, 2], 2, 1.0),
        ([9, 0, 0], 3, 0.5), ([4, 7, 1], 3, 1.0), ([1, 2, 3], 3, 1.0), ([5, 5, 5], 3, 1.0),
        ([1e-13, 2e-13, 0.5, -1], 2, 1.0),        # pipeline != oracle here
        ([0.0, -0.0, 0.0, -0.0], 2, 1.0),          # signed zeros tie
        ([-0.0, 0.0, 1.0], 2, 1.0),
        ([3.0, 3.0, 3.0, 3.0, 3.0], 5, 0.6),      # exact-tie nucleus, fsum exactly 0.6?
        ([1.0], 1, 0.3), ([1.0], 1, 1.0),
    ]
    out = []
    for row, k, p in cases:
        r = np.array(row, dtype=np.float32)
        keep = ref_keep(r, k, p)
        out.append({"row": [float(v) for v in r], "row_bits": r.view(np.uint32).tolist(),
                    "k": k, "p": p, "keep": keep.astype(int).tolist()})
    rng = np.random.default_rng(8)
    for _ in range(20):  # test_pipeline.py:44-52 style
        r = rng.normal(size=503).astype(np.float32)
        k = int(rng.integers(1, 504))
        out.append({"row_bits": r.view(np.uint32).tolist(), "k": k, "p": 1.0,
                    "keep": ref_keep(r, k, 1.0).astype(int).tolist()})
    rng = np.random.default_rng(10)
    for _ in range(20):  # test_pipeline.py:96-102
        r = rng.normal(size=517).astype(np.float32)
        p = float(rng.uniform(0.01, 0.999))
        out.append({"row_bits": r.view(np.uint32).tolist(), "k": 517, "p": p,
                    "keep": ref_keep(r, 517, p).astype(int).tolist()})
    rng = np.random.default_rng(12)
    for _ in range(20):  # test_pipeline.py:131-139
        r = rng.normal(size=251).astype(np.float32)
        k = int(rng.integers(1, 252))
        p = float(rng.uniform(0.01, 0.999))
        out.append({"row_bits": r.view(np.uint32).tolist(), "k": k, "p": p,
                    "keep": ref_keep(r, k, p).astype(int).tolist()})
    for c in out:
        c.pop("row", None)
    with open(os.path.join(HERE, "kats.json"), "w") as fh:
        json.dump(out, fh)
    print("kats:", len(out))


def exhaustive():
    """Criterion-2 style exhaustive small rows (test_acceptance.py:82-110)."""
    rows, ks, ps, trip = [], [], [], []
    for v in range(1, 9):
        for vals in itertools.product((0.0, 1.0, 2.0), repeat=v):
            r = np.zeros(8, dtype=np.float32)
            r[:v] = vals
            for k in range(1, v + 1):
                keep = ref_keep(r[:v], k, 1.0)
                rows.append((v, r.copy())); ks.append(k); ps.append(1.0)
                trip.append(triplet(r[:v], keep))
    for v in range(1, 7):
        for vals in itertools.product((0.0, 0.5, 1.0, 2.0), repeat=v):
            r = np.zeros(8, dtype=np.float32)
            r[:v] = vals
            for p10 in range(1, 10):
                p = p10 / 10.0
                keep = ref_keep(r[:v], v, p)
                rows.append((v, r.copy())); ks.append(v); ps.append(p)
                trip.append(triplet(r[:v], keep))
    np.savez_compressed(
        os.path.join(HERE, "exhaustive.npz"),
        vlen=np.array([v for v, _ in rows], dtype=np.int32),
        rows=np.stack([r for _, r in rows]),
        k=np.array(ks, dtype=np.int64), p=np.array(ps, dtype=np.float64),
        zb=np.array([t[0] for t in trip], dtype=np.uint32),
        cut=np.array([t[1] for t in trip], dtype=np.int64),
        count=np.array([t[2] for t in trip], dtype=np.int64))
    print("exhaustive:", len(rows))


def corpus():
    """Acceptance-style corpus (test_acceptance.py:22-62) at test-friendly sizes."""
    kinds = ("gaussian", "quantized", "uniform", "gaussian_outliers")
    vocabs = (7, 8, 1000, 4096, 32768)
    rows_per = {7: 24, 8: 24, 1000: 16, 4096: 8, 32768: 4}
    data = {}
    meta = []
    for ki, kind in enumerate(kinds):
        for vi, vocab in enumerate(vocabs):
            b = rows_per[vocab]
            kw = {"m": min(50, vocab)} if kind == "gaussian_outliers" else {}
            seed = 1 + ki * 100 + vi
            x = synth(kind, b, vocab, seed, **kw)
            ref_x = sigmatop.synth_batch(kind, b, vocab, seed=seed, **kw).values
            assert np.array_equal(x.view(np.uint32), ref_x.view(np.uint32)), "synth drift"
            rng = np.random.default_rng(vocab)
            cells = []
            for k in sorted({min(k, vocab) for k in (1, 10, 50, vocab - 1, vocab)}):
                if k >= 1:
                    cells.append((f"k={k}", np.full(b, k), np.full(b, 1.0)))
            for p in (0.1, 0.7, 0.9, 0.95, 1.0):
                cells.append((f"p={p}", np.full(b, vocab), np.full(b, p)))
            cells.append(("combined", np.full(b, min(50, vocab)), np.full(b, 0.9)))
            cells.append(("rand", rng.integers(1, vocab + 1, size=b),
                          np.clip(rng.random(b), 1e-12, 1.0 - 1e-12)))
            for label, kk, pp in cells:
                kk = kk.astype(np.int64)
                pp = pp.astype(np.float64)
                trip = np.array([triplet(x[i], ref_keep(x[i], kk[i], pp[i])) for i in range(b)],
                                dtype=np.int64)
                met = ref_metrics(x, kk, pp)
                key = f"{kind}|{vocab}|{label}"
                data[key + "|k"] = kk
                data[key + "|p"] = pp
                data[key + "|trip"] = trip
                for mk, mv in met.items():
                    data[key + "|" + mk] = mv
                meta.append({"key": key, "kind": kind, "vocab": vocab, "batch": b, "seed": seed,
                             "kw": kw, "sha256": sha256(x)})
    np.savez_compressed(os.path.join(HERE, "corpus.npz"), **data)
    with open(os.path.join(HERE, "corpus_meta.json"), "w") as fh:
        json.dump(meta, fh)
    print("corpus cells:", len(meta))


def configs():
    """Every BASELINE config, all rows."""
    data = {}
    meta = {}
    for name in ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5"):
        t0 = time.time()
        x, k, p, dtype = config_inputs(name)
        trip = np.array([triplet(x[i], ref_keep(x[i], k[i], p[i])) for i in range(x.shape[0])],
                        dtype=np.int64)
        data[name + "|trip"] = trip
        data[name + "|k"] = k
        data[name + "|p"] = p
        nmet = min(x.shape[0], 64)
        met = ref_metrics(x[:nmet], k[:nmet], p[:nmet])
        for mk, mv in met.items():
            data[name + "|" + mk] = mv
        meta[name] = {"sha256": sha256(x), "dtype": dtype, "shape": list(x.shape),
                      "metric_rows": nmet}
        print(name, x.shape, f"{time.time() - t0:.1f}s", "mean kept", trip[:, 2].mean())
    np.savez_compressed(os.path.join(HERE, "configs.npz"), **data)
    with open(os.path.join(HERE, "configs_meta.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


ABLATIONS = {  # Table 3 runs of cli.py:157-166 that change the pipeline's configuration
    "C": dict(search_kind="quaternary", duplication_handling_enabled=False),
    "D": dict(search_kind="binary"),
    "E": dict(search_kind="binary", duplication_handling_enabled=False),
    "F": dict(search_kind="quaternary", force_fallback=True),
    "H": dict(search_kind="quaternary", sigma_trunc_enabled=False),
}


def ablation():
    """The reference PIPELINE's own outputs (sigmatop.run_batch, engine.py:82-113) under the
    ablation configurations of Table 3 (cli.py:157-166).  dup_handling=False (runs C, E) changes the
    answer — the whole boundary cluster is kept at each stage (pipeline.py:47-57) — so those
    kept sets come from the pipeline, not the oracle; D / F / H must equal the oracle."""
    data, meta = {}, []
    for ki, kind in enumerate(("gaussian", "quantized")):
        for vi, vocab in enumerate((1000, 4096, 32768)):
            b = {1000: 16, 4096: 8, 32768: 4}[vocab]
            seed = 500 + ki * 10 + vi
            x = synth(kind, b, vocab, seed)
            rng = np.random.default_rng(seed)
            cells = [("k=10", np.full(b, 10), np.full(b, 1.0)), ("k=50", np.full(b, 50), np.full(b, 1.0)),
                     ("p=0.7", np.full(b, vocab), np.full(b, 0.7)), ("p=0.9", np.full(b, vocab), np.full(b, 0.9)),
                     ("combined", np.full(b, 50), np.full(b, 0.9)),
                     ("rand", rng.integers(1, min(vocab, 1024) + 1, size=b), rng.uniform(0.3, 0.99, b))]
            for label, kk, pp in cells:
                kk, pp = kk.astype(np.int64), pp.astype(np.float64)
                key = f"{kind}|{vocab}|{label}"
                data[key + "|k"], data[key + "|p"] = kk, pp
                for run, cfg in ABLATIONS.items():
                    outs, _ = run_batch(LogitBatch(x), TruncTargets(kk, pp), EngineConfig(**cfg))
                    trip = np.array([triplet(x[i], ~np.isneginf(outs[i])) for i in range(b)], dtype=np.int64)
                    data[key + "|" + run] = trip
                meta.append({"key": key, "kind": kind, "vocab": vocab, "batch": b, "seed": seed, "kw": {},
                             "sha256": sha256(x)})
    np.savez_compressed(os.path.join(HERE, "ablation.npz"), **data)
    with open(os.path.join(HERE, "ablation_meta.json"), "w") as fh:
        json.dump({"runs": ABLATIONS, "cells": meta}, fh)
    print("ablation cells:", len(meta), "x", len(ABLATIONS), "runs")


if __name__ == "__main__":
    which = sys.argv[1:] or ["kats", "exhaustive", "corpus", "configs"]
    for w in which:
        globals()[w]()
