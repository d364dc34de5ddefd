"""GPU: the bf16 top-p-only kernel (qrita_topp16: two-CTA clusters, direct-mapped 16-bit key
histograms) against the oracle — heavy ties, keep-all rows, index-only and in-place output,
duplicate-handling ablation, and the rows it hands back to the fused kernel (non-finite logits,
a value repeated more than 65535 times in a segment)."""
import numpy as np
import pytest
import torch

import paper_2602_01518_b200 as Q
from oracle.qrita_oracle import oracle_batch, oracle_keep_row_nodup
from oracle.synth import bf16_bits_to_f32, to_bf16_bits
from tests import golden_io as G

pytestmark = pytest.mark.gpu


def bf16_rows(b, v, seed, quant=True):
    r = np.random.default_rng(seed)
    x = r.normal(0, 1, (b, v)).astype(np.float32) * r.uniform(0.5, 4, (b, 1)).astype(np.float32)
    if quant:
        neg = x < 0
        x[neg] = np.round(4 * x[neg]) / 4
    return bf16_bits_to_f32(to_bf16_bits(x))


def run(x, k, p, **kw):
    xt = torch.from_numpy(x).cuda().to(torch.bfloat16)
    kc = torch.zeros(x.shape[0], dtype=torch.int32, device="cuda")
    met = Q.ops.metrics_buffer(x.shape[0], xt.device)
    out = Q.topk_topp(xt, torch.from_numpy(k).cuda(), torch.from_numpy(p).cuda(), kept_count=kc, metrics=met,
                      check=True, **kw)
    return out.float().cpu().numpy(), kc.cpu().numpy(), Q.ops.decode_metrics(met)


@pytest.mark.parametrize("v", [4096, 8200, 65536, 151936, 262144])
def test_topp_only_rows_vs_oracle(cuda_device, v):
    x = bf16_rows(12, v, v)
    k = np.full(12, v, np.int64)
    p = np.array([0.95, 0.5, 0.999, 0.01, 0.9, 0.7, 1 - 2 ** -50, 0.3, 0.99, 0.6, 0.8, 0.97])
    got, kc, met = run(x, k, p)
    want, cnt = oracle_batch(x, k, p)
    assert G.same_bits(got, want).all()
    assert np.array_equal(kc, cnt)
    assert all(m["row_passes"] == 2 for m in met), [m["row_passes"] for m in met]


def test_mixed_modes_bf16_batch(cuda_device):
    v = 32768
    x = bf16_rows(40, v, 3)
    r = np.random.default_rng(4)
    k = r.integers(1, 1025, 40).astype(np.int64)
    p = r.uniform(0.3, 0.99, 40)
    k[::2] = v           # top-p only rows -> qrita_topp16
    p[1::4] = 1.0        # top-k only rows -> fused
    k[3], p[3] = v, 1.0  # pass-through
    got, kc, _ = run(x, k, p)
    want, cnt = oracle_batch(x, k, p)
    assert G.same_bits(got, want).all() and np.array_equal(kc, cnt)


def test_index_only_inplace_and_nodup(cuda_device):
    v = 16384
    x = bf16_rows(6, v, 9)
    k = np.full(6, v, np.int64)
    p = np.linspace(0.4, 0.98, 6)
    want, cnt = oracle_batch(x, k, p)
    xt = torch.from_numpy(x).cuda().to(torch.bfloat16)
    idx, kc = Q.topk_topp_indices(xt, torch.from_numpy(k).cuda(), torch.from_numpy(p).cuda(), check=True)
    idx, kc = idx.cpu().numpy(), kc.cpu().numpy()
    assert np.array_equal(kc, cnt)
    for i in range(6):
        assert np.array_equal(np.sort(idx[i, :kc[i]]), np.nonzero(~np.isneginf(want[i]))[0])
    y = xt.clone()
    Q.topk_topp(y, torch.from_numpy(k).cuda(), torch.from_numpy(p).cuda(), inplace=True, check=True)
    assert G.same_bits(y.float().cpu().numpy(), want).all()
    got, _, _ = run(x, k, p, flags=Q.TruncFlags(dup_handling=False))
    for i in range(6):
        assert np.array_equal(~np.isneginf(got[i]), oracle_keep_row_nodup(x[i], v, float(p[i])))


def test_rows_handed_back_to_the_fused_kernel(cuda_device):
    v = 150000
    x = bf16_rows(3, v, 5)
    x[1, :] = 0.5            # 75000 copies of one value per segment: counter overflow
    x[2, 777] = np.nan       # non-finite: the fused kernel reports it
    k = np.full(3, v, np.int64)
    p = np.array([0.9, 0.6, 0.9])
    xt = torch.from_numpy(x).cuda().to(torch.bfloat16)
    with pytest.raises(ValueError, match="NaN logit at row 2, col 777"):
        Q.topk_topp(xt, torch.from_numpy(k).cuda(), torch.from_numpy(p).cuda(), check=True)
    got, kc, _ = run(x[:2], k[:2], p[:2])
    want, cnt = oracle_batch(x[:2], k[:2], p[:2])
    assert G.same_bits(got, want).all() and np.array_equal(kc, cnt)


def test_cfg3_metrics_match_reference(cuda_device):
    x, k, p, _, trip, mets = G.config("cfg3")
    got, kc, met = run(x, k, p)
    assert G.same_bits(got, G.masked_from_trip(x, trip)).all()
    n = mets["outlier_count"].shape[0]
    assert [m["outlier_count"] for m in met[:n]] == mets["outlier_count"].tolist()
    assert [m["trunc_hit"] for m in met[:n]] == mets["trunc_hit"].astype(int).tolist()
