"""GPU: the LM-head producer fusion (csrc/qrita_lmhead.cu).  The tcgen05 GEMM is checked against a
torch fp32 matmul of the same bf16 operands (tolerance below: fp32 accumulation order differs), the
fused call's logits against the plain GEMM bit for bit, and its kept sets against
topk_topp_indices on those logits and the oracle (oracle.py:70-89) — bit-exact."""
import numpy as np
import pytest
import torch

import paper_2602_01518_b200 as Q
from oracle.qrita_oracle import oracle_batch
from paper_2602_01518_b200.lmhead import lm_head_logits, lm_head_topk_topp

pytestmark = pytest.mark.gpu


def _operands(b, v, d, seed):
    g = torch.Generator(device="cpu").manual_seed(seed)
    h = torch.randn(b, d, generator=g).to(torch.bfloat16).cuda()
    w = (torch.randn(v, d, generator=g) / d ** 0.5).to(torch.bfloat16).cuda()
    return h, w


@pytest.mark.parametrize("b,v,d", [(1, 1000, 64), (8, 4096, 128), (37, 5000, 256), (256, 32000, 512),
                                   (300, 2100, 192)])
def test_logits_match_fp32_matmul(cuda_device, b, v, d):
    h, w = _operands(b, v, d, b + v + d)
    got = lm_head_logits(h, w)
    want = h.float() @ w.float().T
    scale = (h.float().abs() @ w.float().abs().T)
    # |fp32 sum reordering| <= d * 2^-24 * sum |terms|; 4x margin
    tol = 4 * d * 2.0 ** -24 * scale
    assert bool(((got - want).abs() <= tol + 1e-30).all()), float(((got - want).abs() / (scale + 1e-30)).max())


def _kept_sets(idx, cnt):
    idx, cnt = idx.cpu().numpy(), cnt.cpu().numpy()
    return [np.sort(idx[r, :cnt[r]]) for r in range(len(cnt))]


@pytest.mark.parametrize("b,v,d", [(4, 4096, 128), (37, 32000, 256), (130, 9000, 128), (300, 5000, 64),
                                   (9, 1000, 64), (20, 2500, 128), (3, 100, 64), (17, 129, 64)])
def test_fused_kept_sets_exact(cuda_device, b, v, d):
    h, w = _operands(b, v, d, 7 * b + v)
    if b > 5:
        h[5] = 0                                        # an all-tied row (every logit 0)
    rng = np.random.default_rng(b + v)
    k = np.minimum(rng.integers(1, 1025, b), v).astype(np.int64)
    p = rng.uniform(0.3, 0.99, b)
    k[::7] = v                                          # top-p only (whole row)
    p[1::5] = 1.0                                       # top-k only
    if b > 3:
        k[3], p[3] = v, 1.0                             # pass-through
    logits, kidx, kc = lm_head_topk_topp(h, w, torch.from_numpy(k), torch.from_numpy(p), check=True)
    ref = lm_head_logits(h, w)
    assert torch.equal(logits, ref)
    want_idx, want_cnt = Q.topk_topp_indices(ref, torch.from_numpy(k).cuda(), torch.from_numpy(p).cuda())
    got, want = _kept_sets(kidx, kc), _kept_sets(want_idx, want_cnt)
    assert all(np.array_equal(a, c) for a, c in zip(got, want))
    masked, _ = oracle_batch(ref.cpu().numpy(), k, p)
    for r in range(b):
        assert np.array_equal(got[r], np.nonzero(~np.isneginf(masked[r]))[0]), r


def test_fused_forced_fallback_and_binary(cuda_device):
    h, w = _operands(16, 6000, 128, 11)
    k = torch.full((16,), 40, dtype=torch.int64)
    p = torch.full((16,), 0.8, dtype=torch.float64)
    ref = lm_head_logits(h, w)
    want = _kept_sets(*Q.topk_topp_indices(ref, k.cuda(), p.cuda()))
    for fl in (Q.TruncFlags(force_fallback=True), Q.TruncFlags(search="binary"), Q.TruncFlags(use_sigma_trunc=False)):
        _, kidx, kc = lm_head_topk_topp(h, w, k, p, flags=fl)
        assert all(np.array_equal(a, c) for a, c in zip(_kept_sets(kidx, kc), want))


def test_fused_invalid_rows_raise(cuda_device):
    h, w = _operands(4, 1000, 64, 2)
    with pytest.raises(ValueError):
        lm_head_topk_topp(h, w, torch.tensor([5, 0, 5, 5]), 0.9, check=True)
    with pytest.raises(ValueError):
        lm_head_logits(h[:, :60].contiguous(), w[:, :60].contiguous())


def test_fused_metrics_match_the_truncation_path(cuda_device):
    """The fused epilogue plans from the same (bit-identical) sample logits and counts outliers with
    the same predicate as the streaming pass, so the reference's per-row metrics agree."""
    b, v, d = 24, 20000, 128
    h, w = _operands(b, v, d, 99)
    rng = np.random.default_rng(4)
    k = torch.from_numpy(rng.integers(1, 600, b).astype(np.int64))
    p = torch.from_numpy(rng.uniform(0.4, 0.99, b))
    mf = Q.ops.metrics_buffer(b, "cuda")
    logits, kidx, kc = lm_head_topk_topp(h, w, k, p, metrics=mf)
    mr = Q.ops.metrics_buffer(b, "cuda")
    Q.topk_topp_indices(logits, k.cuda(), p.cuda(), metrics=mr)
    got, want = Q.ops.decode_metrics(mf), Q.ops.decode_metrics(mr)
    for r in range(b):
        for key in ("trunc_hit", "outlier_count", "fallback_used", "kept_count"):
            assert got[r][key] == want[r][key], (r, key, got[r][key], want[r][key])


def test_fused_compact_kept_lists(cuda_device):
    h, w = _operands(12, 9000, 128, 5)
    k = torch.tensor([5, 1000, 64, 999, 1, 300, 17, 1000, 2, 800, 50, 1000])
    p = torch.full((12,), 0.9, dtype=torch.float64)
    logits, kidx, kc = lm_head_topk_topp(h, w, k, p, k_cap=1000)
    assert kidx.shape == (12, 1000)
    want = _kept_sets(*Q.topk_topp_indices(logits, k.cuda(), p.cuda()))
    assert all(np.array_equal(a, c) for a, c in zip(_kept_sets(kidx, kc), want))
    with pytest.raises(ValueError):
        lm_head_topk_topp(h, w, k, p, k_cap=999)


def test_capi_binding_as_documented(cuda_device):
    """The INTEGRATION.md ctypes binding of qrita_lmhead_topk_topp, argument for argument."""
    import ctypes
    from paper_2602_01518_b200 import _native as N
    lib = N.load()
    B, V, d = 6, 3000, 128
    hidden, weight = _operands(B, V, d, 21)
    kt = torch.tensor([5, 50, 300, 1, 999, 64], dtype=torch.int64, device="cuda")
    pt = torch.tensor([0.9, 0.5, 1.0, 1.0, 0.95, 0.8], dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    nbytes = lib.qrita_lmhead_workspace_bytes(B, V)
    ws = torch.zeros(nbytes + 256, dtype=torch.uint8, device="cuda"); wsp = (ws.data_ptr() + 255) & ~255
    logits = torch.empty(B, V, device="cuda"); kidx = torch.empty(B, V, dtype=torch.int32, device="cuda")
    kcnt = torch.empty(B, dtype=torch.int32, device="cuda")
    rc = lib.qrita_lmhead_topk_topp(hidden.data_ptr(), d, weight.data_ptr(), d, B, V, d, kt.data_ptr(),
                                    pt.data_ptr(), logits.data_ptr(), V, kidx.data_ptr(), V, kcnt.data_ptr(),
                                    None, wsp, nbytes, 0, st)
    assert rc == N.OK
    row, col = ctypes.c_int(), ctypes.c_int()
    assert lib.qrita_get_status(wsp, B, ctypes.byref(row), ctypes.byref(col), st) == N.OK
    want = _kept_sets(*Q.topk_topp_indices(logits, kt, pt))
    assert all(np.array_equal(a, c) for a, c in zip(_kept_sets(kidx, kcnt), want))
