"""GPU: row-sharded execution (topk_topp_sharded / run_batch(devices=...)) is bit-exact against the
reference's golden answers.  Only one GPU is available to the tests, so the device list repeats
device 0: every block still gets its own stream, workspace and host-pipeline scratch."""
import numpy as np
import pytest
import torch

import paper_2602_01518_b200 as Q
from paper_2602_01518_b200.sharded import topk_topp_sharded
from tests import golden_io as G

pytestmark = pytest.mark.gpu


def _check(x, got, trip, label):
    want = G.masked_from_trip(x, trip)
    bad = np.nonzero(~G.same_bits(got, want).all(axis=1))[0]
    assert bad.size == 0, f"{label}: {bad.size} rows differ, first {bad[:5]}"


def test_sharded_host_cfg4_two_blocks(cuda_device):
    x, k, p, _, trip, _ = G.config("cfg4")
    xh = torch.from_numpy(x).pin_memory()
    kept = torch.zeros(x.shape[0], dtype=torch.int32)
    out = topk_topp_sharded(xh, torch.from_numpy(k), torch.from_numpy(p), devices=[0, 0], kept_count=kept)
    assert not out.is_cuda
    _check(x, out.numpy(), trip, "cfg4 host [0,0]")
    assert np.array_equal(kept.numpy(), trip[:, 2])


def test_sharded_device_cfg2_three_blocks(cuda_device):
    x, k, p, _, trip, _ = G.config("cfg2")
    xt = torch.from_numpy(x).cuda()
    met = Q.ops.metrics_buffer(x.shape[0], xt.device)
    out = topk_topp_sharded(xt, torch.from_numpy(k), torch.from_numpy(p), devices=[0, 0, 0], metrics=met)
    assert out.is_cuda
    torch.cuda.synchronize()
    _check(x, out.cpu().numpy(), trip, "cfg2 device [0,0,0]")
    assert [m["kept_count"] for m in Q.ops.decode_metrics(met)] == trip[:, 2].tolist()


def test_sharded_numpy_pageable_and_errors(cuda_device):
    x, k, p, _, trip, _ = G.config("cfg2")
    out = topk_topp_sharded(x[:37], k[:37], p[:37], devices=[0, 0])
    _check(x[:37], out.numpy(), trip[:37], "cfg2 numpy [0,0]")
    bad = x[:20].copy()
    bad[13, 77] = np.nan
    with pytest.raises(ValueError, match="NaN logit at row 13, col 77"):
        topk_topp_sharded(bad, k[:20], p[:20], devices=[0, 0])


def test_run_batch_numpy_host_pipeline(cuda_device):
    x, k, p, _, trip, mets = G.config("cfg2")
    outs, rep = Q.run_batch(Q.LogitBatch(x), Q.TruncTargets(k, p), Q.EngineConfig())
    assert isinstance(outs, np.ndarray) and outs.dtype == np.float32
    _check(x, outs, trip, "run_batch cfg2")
    n = len(mets["trunc_hit"])
    assert [m.trunc_hit for m in rep.per_row[:n]] == mets["trunc_hit"].astype(bool).tolist()
    assert [m.outlier_count for m in rep.per_row[:n]] == mets["outlier_count"].tolist()
    outs2, rep2 = Q.run_batch(Q.LogitBatch(x), Q.TruncTargets(k, p), Q.EngineConfig(), devices=[0, 0])
    assert G.same_bits(outs, outs2).all() and rep2.hit_rate == rep.hit_rate


def test_run_batch_errors_match_reference_text(cuda_device):
    vals = np.zeros((3, 64), dtype=np.float32)
    vals[2, 5] = np.inf
    with pytest.raises(ValueError, match=r"^invalid batch: non-finite logit at row 2, col 5$"):
        Q.run_batch(Q.LogitBatch(vals), Q.TruncTargets.uniform(3, 4, 0.5), Q.EngineConfig())
    vals[2, 5] = 0.0
    with pytest.raises(ValueError, match=r"row 1: k out of range"):
        Q.run_batch(Q.LogitBatch(vals), Q.TruncTargets(np.array([1, 65, 2]), np.full(3, 0.5)), Q.EngineConfig())
