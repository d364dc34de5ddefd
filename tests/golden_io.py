"""Loaders for the golden fixtures written by tests/golden/make_golden.py (reference-generated)."""
from __future__ import annotations

import json
import os

import numpy as np

from oracle.qrita_oracle import mask_from_boundary
from oracle.synth import config_inputs, sha256, synth

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def kats():
    with open(os.path.join(GOLDEN, "kats.json")) as fh:
        cases = json.load(fh)
    out = []
    for c in cases:
        row = np.array(c["row_bits"], dtype=np.uint32).view(np.float32)
        out.append((row, int(c["k"]), float(c["p"]), np.array(c["keep"], dtype=bool)))
    return out


def exhaustive():
    z = np.load(os.path.join(GOLDEN, "exhaustive.npz"))
    return {k: z[k] for k in z.files}


def corpus():
    """Yields (key, x, k, p, trip, metrics) per cell, inputs regenerated from seeds."""
    with open(os.path.join(GOLDEN, "corpus_meta.json")) as fh:
        meta = json.load(fh)
    z = np.load(os.path.join(GOLDEN, "corpus.npz"))
    cache = {}
    for m in meta:
        sk = (m["kind"], m["vocab"], m["batch"], m["seed"])
        if sk not in cache:
            x = synth(m["kind"], m["batch"], m["vocab"], m["seed"], **m["kw"])
            assert sha256(x) == m["sha256"], f"input drift for {m['key']}"
            cache[sk] = x
        key = m["key"]
        mets = {f: z[key + "|" + f] for f in ("trunc_hit", "outlier_count", "outlier_prob_sum",
                                              "fallback_used")}
        yield key, cache[sk], z[key + "|k"], z[key + "|p"], z[key + "|trip"], mets


_CFG_CACHE = {}


def config(name: str):
    """(x f32 [B,V], k, p, dtype, trip [B,3], metrics dict over the first metric_rows rows)."""
    if name not in _CFG_CACHE:
        with open(os.path.join(GOLDEN, "configs_meta.json")) as fh:
            meta = json.load(fh)[name]
        x, k, p, dtype = config_inputs(name)
        assert sha256(x) == meta["sha256"], f"input drift for {name}"
        z = np.load(os.path.join(GOLDEN, "configs.npz"))
        assert np.array_equal(z[name + "|k"], k) and np.array_equal(z[name + "|p"], p)
        mets = {f: z[name + "|" + f] for f in ("trunc_hit", "outlier_count", "outlier_prob_sum",
                                               "fallback_used")}
        _CFG_CACHE[name] = (x, k, p, dtype, z[name + "|trip"], mets)
    return _CFG_CACHE[name]


def keep_from_trip(row, trip) -> np.ndarray:
    return mask_from_boundary(row, int(trip[0]), int(trip[1]))


def masked_from_trip(x: np.ndarray, trip: np.ndarray) -> np.ndarray:
    out = np.full_like(x, -np.inf)
    for i in range(x.shape[0]):
        keep = keep_from_trip(x[i], trip[i])
        out[i, keep] = x[i, keep]
    return out


def same_bits(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Elementwise bit equality, -inf == -inf (verify_batch's rule, engine.py:129)."""
    a = np.asarray(a, dtype=np.float32)
    b = np.asarray(b, dtype=np.float32)
    return (a.view(np.uint32) == b.view(np.uint32)) | (np.isneginf(a) & np.isneginf(b))


def ablation():
    """Yields (key, x, k, p, {run: trip}) per cell of tests/golden/ablation.npz (the reference pipeline
    under Table 3's ablation configurations), inputs regenerated from seeds."""
    with open(os.path.join(GOLDEN, "ablation_meta.json")) as fh:
        meta = json.load(fh)
    z = np.load(os.path.join(GOLDEN, "ablation.npz"))
    runs = list(meta["runs"])
    cache = {}
    for m in meta["cells"]:
        sk = (m["kind"], m["vocab"], m["batch"], m["seed"])
        if sk not in cache:
            x = synth(m["kind"], m["batch"], m["vocab"], m["seed"])
            assert sha256(x) == m["sha256"], f"input drift for {m['key']}"
            cache[sk] = x
        key = m["key"]
        yield key, cache[sk], z[key + "|k"], z[key + "|p"], {r: z[key + "|" + r] for r in runs}


ABLATION_FLAGS = {  # Table 3 run -> this build's TruncFlags keyword arguments
    "C": dict(dup_handling=False),
    "D": dict(search="binary"),
    "E": dict(search="binary", dup_handling=False),
    "F": dict(force_fallback=True),
    "H": dict(use_sigma_trunc=False),
}
