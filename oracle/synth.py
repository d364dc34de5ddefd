"""Deterministic input generators for tests and benchmarks — TEST INFRASTRUCTURE ONLY.

Inputs are regenerated from seeds instead of being stored.  The gaussian / quantized / uniform /
gaussian_outliers laws follow the reference's `synth_batch` (engine.py:139-180) draw for draw, so a
seed produces the same float32 matrix here as in the reference (checked by sha256 in the golden
fixtures).  The BASELINE configs are built on top.
"""
from __future__ import annotations

import hashlib

import numpy as np


def synth(kind: str, batch: int, vocab: int, seed: int, **kw) -> np.ndarray:
    """float32 [batch, vocab] matrix; same random stream as sigmatop.engine.synth_batch."""
    rng = np.random.default_rng(seed)
    if kind == "gaussian":
        vals = rng.normal(kw.get("mu0", 0.0), kw.get("sigma0", 1.0), size=(batch, vocab))
    elif kind == "gaussian_outliers":
        m = int(kw.get("m", 50))
        mag = kw.get("magnitude", 12.0)
        vals = rng.normal(0.0, 1.0, size=(batch, vocab))
        for r in range(batch):
            cols = rng.choice(vocab, size=m, replace=False)
            vals[r, cols] = mag + rng.random(m)
    elif kind == "quantized":
        g = int(kw.get("g", 16))
        levels = np.linspace(-3.0, 3.0, g)
        z = np.clip(rng.normal(0.0, 1.0, size=(batch, vocab)), -3, 3)
        if batch * vocab <= 1 << 20:
            vals = levels[np.argmin(np.abs(z[..., None] - levels), axis=-1)]
        else:
            vals = levels[np.clip(np.round((z + 3.0) / 6.0 * (g - 1)).astype(np.int64), 0, g - 1)]
    elif kind == "uniform":
        vals = rng.uniform(kw.get("low", 0.0), kw.get("high", 1.0), size=(batch, vocab))
    else:
        raise ValueError(f"unknown kind {kind!r}")
    return vals.astype(np.float32)


def to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """float32 -> bfloat16 bit patterns, round to nearest even (as torch's .to(torch.bfloat16))."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    rounding = ((b >> 16) & 1) + 0x7FFF
    out = ((b + rounding) >> 16).astype(np.uint16)
    return out


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32)


def config_inputs(name: str):
    """(logits f32 [B,V] (bf16-representable for cfg3), k int64[B], p float64[B], dtype) per
    BASELINE config."""
    if name == "cfg1":
        x = synth("gaussian", 1, 32000, seed=0)
        return x, np.full(1, 50, np.int64), np.full(1, 0.9), "f32"
    if name == "cfg2":
        x = synth("gaussian", 256, 128256, seed=1)
        r = np.random.default_rng(42)
        return x, r.integers(1, 1025, 256).astype(np.int64), r.uniform(0.5, 0.99, 256), "f32"
    if name == "cfg3":
        r = np.random.default_rng(3)
        x = r.normal(0.0, 1.0, (64, 151936)).astype(np.float32)
        neg = x < 0
        x[neg] = np.round(4.0 * x[neg]) / 4.0
        x = bf16_bits_to_f32(to_bf16_bits(x))
        return x, np.full(64, 151936, np.int64), np.full(64, 0.95), "bf16"
    if name == "cfg4":
        x = synth("gaussian", 1024, 262144, seed=4)
        r = np.random.default_rng(44)
        return x, r.integers(1, 1025, 1024).astype(np.int64), r.uniform(0.5, 0.99, 1024), "f32"
    if name == "cfg5":
        x = synth("gaussian", 128, 262144, seed=5)
        r = np.random.default_rng(55)
        return x, r.integers(1, 1025, 128).astype(np.int64), r.uniform(0.5, 0.99, 128), "f32"
    raise ValueError(name)


def sha256(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
