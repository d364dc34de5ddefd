"""CPU: pin the oracle restatement (oracle/qrita_oracle.py) to the reference's own answers.

Golden vectors come from tests/golden/make_golden.py, which ran the reference package itself.
"""
import numpy as np
import pytest

from oracle.qrita_oracle import (boundary_of_mask, crossing_margin, mask_from_boundary,
                                 oracle_batch, oracle_keep_row, oracle_keep_row_nodup)
from oracle.synth import bf16_bits_to_f32, to_bf16_bits
from tests import golden_io as G


def test_kats_match_reference():
    cases = G.kats()
    assert len(cases) >= 70
    for row, k, p, keep in cases:
        assert np.array_equal(oracle_keep_row(row, k, p), keep), (row[:8], k, p)


def test_tiny_logit_tie_case_follows_oracle_not_pipeline():
    # the reference pipeline's eq_eps disagrees with its oracle here; we follow the oracle.
    row = np.array([1e-13, 2e-13, 0.5, -1], dtype=np.float32)
    keep = oracle_keep_row(row, 2, 1.0)
    assert keep.tolist() == [False, True, True, False]


def test_exhaustive_small_rows():
    z = G.exhaustive()
    n = z["k"].shape[0]
    idx = np.arange(n) if n < 40000 else np.random.default_rng(0).choice(n, 40000, replace=False)
    for i in idx:
        v = int(z["vlen"][i])
        row = z["rows"][i, :v]
        keep = oracle_keep_row(row, int(z["k"][i]), float(z["p"][i]))
        want = mask_from_boundary(row, int(z["zb"][i]), int(z["cut"][i]))
        assert np.array_equal(keep, want), (row, z["k"][i], z["p"][i])


def test_acceptance_corpus():
    cells = 0
    for key, x, k, p, trip, _ in G.corpus():
        if x.shape[1] > 5000:
            continue  # the 32768-wide cells are covered on the GPU
        for i in range(x.shape[0]):
            keep = oracle_keep_row(x[i], int(k[i]), float(p[i]))
            assert np.array_equal(keep, G.keep_from_trip(x[i], trip[i])), (key, i)
        cells += 1
    assert cells >= 150


@pytest.mark.parametrize("name,rows", [("cfg1", 1), ("cfg2", 24), ("cfg3", 4), ("cfg5", 8)])
def test_configs(name, rows):
    x, k, p, dtype, trip, _ = G.config(name)
    for i in range(rows):
        keep = oracle_keep_row(x[i], int(k[i]), float(p[i]))
        assert np.array_equal(keep, G.keep_from_trip(x[i], trip[i])), (name, i)


def test_boundary_encoding_roundtrip():
    rng = np.random.default_rng(5)
    for _ in range(50):
        row = np.round(rng.normal(size=200) * 2).astype(np.float32)
        k = int(rng.integers(1, 201))
        keep = oracle_keep_row(row, k, 1.0)
        zb, cut, cnt = boundary_of_mask(row, keep)
        assert cnt == k
        assert np.array_equal(mask_from_boundary(row, zb, cut), keep)


def test_oracle_batch_and_margin():
    rng = np.random.default_rng(6)
    x = rng.normal(size=(4, 300)).astype(np.float32)
    out, cnt = oracle_batch(x, [5, 300, 300, 20], [1.0, 0.5, 1.0, 0.9])
    assert cnt.tolist()[0] == 5 and cnt.tolist()[2] == 300
    assert np.array_equal(out[2], x[2])
    assert crossing_margin(x[1], 300, 0.5) > 1e-13


def test_bf16_rounding_matches_torch():
    import torch
    x = np.random.default_rng(7).normal(size=10000).astype(np.float32) * 3
    ours = to_bf16_bits(x)
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(ours, ref)
    assert np.array_equal(bf16_bits_to_f32(ours), torch.from_numpy(x).to(torch.bfloat16).float().numpy())


def test_ablation_goldens_pin_the_oracles():
    """Table 3 ablations: runs D / F / H (binary search, forced fallback, no sigma) leave the answer
    unchanged (the oracle's); runs C / E (no duplicate handling) follow the pipeline's whole-cluster
    rule, restated by oracle_keep_row_nodup."""
    n = 0
    for key, x, k, p, runs in G.ablation():
        for i in range(x.shape[0]):
            exact = oracle_keep_row(x[i], int(k[i]), float(p[i]))
            nodup = oracle_keep_row_nodup(x[i], int(k[i]), float(p[i]))
            for run, trip in runs.items():
                want = G.keep_from_trip(x[i], trip[i])
                got = nodup if run in ("C", "E") else exact
                assert np.array_equal(got, want), (key, run, i)
                n += 1
    assert n >= 5 * 150
