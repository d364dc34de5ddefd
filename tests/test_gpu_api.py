"""GPU: the drop-in primitives beyond run_batch — sigma_trunc's row_stats / gather_outliers, the
search and oracle entry points, QRTL straight to HBM, Table 3's ablation front-end and table
generation — against numpy's own arithmetic (the reference's) and the oracle."""
import numpy as np
import pytest
import torch

import paper_2602_01518_b200 as Q
from oracle.qrita_oracle import oracle_keep_row
from paper_2602_01518_b200 import cli
from tests import golden_io as G

pytestmark = pytest.mark.gpu


def np_row_stats(row, s=4096):
    prefix = np.asarray(row[:s], dtype=np.float64)
    mu = float(prefix.mean())
    var = float((prefix * prefix).mean()) - mu * mu
    return mu, float(np.sqrt(max(var, 0.0)))


@pytest.mark.parametrize("v,s", [(7, 4096), (129, 4096), (32000, 4096), (32000, 1000), (128256, 6000),
                                 (5000, 5000)])
def test_row_stats_bit_identical_to_numpy(cuda_device, v, s):
    rng = np.random.default_rng(v + s)
    for _ in range(3):
        row = (rng.normal(size=v) * rng.uniform(0.1, 30)).astype(np.float32)
        got = Q.row_stats(row, s)
        mu, sigma = np_row_stats(row, s)
        assert (got.mu, got.sigma, got.sample_size) == (mu, sigma, min(s, v))


def test_gather_outliers_and_hit(cuda_device):
    row = np.random.default_rng(3).normal(size=20000).astype(np.float32)
    st = Q.row_stats(row)
    d = Q.lookup_delta_topk(50, row.shape[0])
    o = Q.gather_outliers(row, st, d)
    t = Q.threshold_from(st, d).t
    want = row.astype(np.float64)[row.astype(np.float64) > t]
    assert np.array_equal(o.values, want) and o.count == want.size
    assert o.row_max == float(row.max()) and o.row_min == float(row.min())
    assert Q.is_hit(o, k=50) == (want.size > 50)
    op = Q.gather_outliers(row, st, Q.lookup_delta_topp(0.9), mode="topp")
    assert 0.0 < op.prob_sum < 1.0


def test_search_entry_points_exact(cuda_device):
    rng = np.random.default_rng(5)
    for _ in range(20):
        vals = np.round(rng.normal(size=300) * 3).astype(np.float64)
        k = int(rng.integers(1, 300))
        r = Q.quaternary_topk(vals, k)
        zs = np.sort(vals)[::-1]
        assert r.z_dup == zs[k - 1] and r.n_dup == int((vals == zs[k - 1]).sum())
        assert r.n_above >= k and r.n_above - r.n_dup < k
        assert Q.binary_topk(vals, k).z_dup == r.z_dup
    assert Q.quaternary_topk(np.full(5, 2.0), 3).ties_only
    probs = np.array([0.4, 0.2, 0.2, 0.1, 0.1])
    r = Q.quaternary_topp(probs, 0.7)
    assert (r.p_mn, r.n_dup, r.n_keep) == (0.2, 2, 2)
    with pytest.raises(ValueError):
        Q.quaternary_topp(probs, 1.0)


def test_oracle_entry_points(cuda_device):
    rng = np.random.default_rng(6)
    row = np.round(rng.normal(size=3000) * 4).astype(np.float32) / 4
    for k, p in ((7, 1.0), (3000, 0.8), (200, 0.6)):
        out = Q.oracle_topk_topp(row, k, p)
        keep = oracle_keep_row(row, k, p)
        assert np.array_equal(~np.isneginf(out.masked_row), keep) and out.kept_count == keep.sum()
    assert Q.oracle_topk(row, 5).kept_count == 5
    assert np.array_equal(~np.isneginf(Q.oracle_topp(row, 0.5).masked_row), oracle_keep_row(row, 3000, 0.5))


def test_qrtl_to_device(cuda_device, tmp_path):
    x, k, p, _, trip, _ = G.config("cfg1")
    Q.write_logits(Q.LogitBatch(x), tmp_path / "c.qrtl")
    b = Q.read_logits(tmp_path / "c.qrtl", device="cuda")
    assert b.values.is_cuda and np.array_equal(b.values.cpu().numpy(), x)
    out, rep = Q.run_batch(b, Q.TruncTargets(k, p), Q.EngineConfig())
    assert G.same_bits(out.cpu().numpy(), G.masked_from_trip(x, trip)).all()


def test_cli_run_verify_bench(cuda_device, tmp_path):
    assert cli.main(["verify", "--batch", "8", "--vocab", "3000"]) == cli.EXIT_OK
    assert cli.main(["verify", "--exhaustive", "--vocab", "5"]) == cli.EXIT_OK
    assert cli.main(["run", "--batch", "4", "--vocab", "4096", "--k", "rand", "--p", "rand",
                     "--out", str(tmp_path / "o.qrtl"), "--report", str(tmp_path / "r.csv")]) == cli.EXIT_OK
    assert Q.read_logits(tmp_path / "o.qrtl").values.shape == (4, 4096)
    rc = cli.main(["bench", "--batch", "16", "--vocab", "8192", "--repeats", "3",
                   "--report", str(tmp_path / "b.csv")])
    lines = (tmp_path / "b.csv").read_text().splitlines()
    assert lines[0].endswith(",parity") and len(lines) == 1 + 9
    assert all(line.endswith("bit-exact") for line in lines[1:]), lines
    assert rc == cli.EXIT_OK


def test_sort_select_sigma_trunc_run_i(cuda_device):
    x, k, p, _, trip, _ = G.config("cfg2")
    b = Q.LogitBatch(x[:16])
    t = Q.TruncTargets(k[:16], p[:16])
    a = Q.sort_select(b, t, use_sigma_trunc=True)
    assert G.same_bits(a, G.masked_from_trip(x[:16], trip[:16])).all()


def test_generate_tables_gpu(cuda_device):
    ek = Q.generate_table_entries("topk", 200_000, 0)
    s = np.sort(np.random.default_rng(0).standard_normal(200_000))[::-1]
    idx = np.minimum(np.ceil(np.arange(1, 201) / 200 * 200_000).astype(np.int64) - 1, 200_000 - 1)
    assert np.array_equal(ek, s[idx])
    ep = Q.generate_table_entries("topp", 200_000, 0)
    exps = np.exp(s - s[0])
    csum = np.cumsum(exps / exps.sum())
    want = s[np.minimum(np.searchsorted(csum, np.arange(1, 201) / 200, side="left"), 200_000 - 1)]
    # the GPU's cumulative sums round differently from numpy's sequential cumsum: an entry may move to
    # the neighbouring sample where two cumulative masses straddle a target within a few ulps
    assert (ep == want).mean() > 0.95 and np.max(np.abs(ep - want)) < 1e-3
    tk, tp = Q.profile_tables(torch.randn(8, 50000, device="cuda"))
    assert abs(tk.entries[100] - 0.0) < 0.05 and tp.kind == "topp"
