"""GPU parity: the B200 kernels (through the C ABI) against the reference's golden answers and the
oracle.  Bar: kept-index sets bit-exact, kept values bit-identical, -inf elsewhere."""
import numpy as np
import pytest
import torch

import paper_2602_01518_b200 as Q
from oracle.qrita_oracle import oracle_keep_row
from oracle.synth import to_bf16_bits
from tests import golden_io as G

pytestmark = pytest.mark.gpu


def run(x, k, p, dtype=torch.float32, **flags):
    xt = torch.from_numpy(np.ascontiguousarray(x)).to("cuda").to(dtype)
    kt = torch.as_tensor(np.asarray(k, dtype=np.int64), device="cuda")
    pt = torch.as_tensor(np.asarray(p, dtype=np.float64), device="cuda")
    kept = torch.zeros(xt.shape[0], dtype=torch.int32, device="cuda")
    met = Q.ops.metrics_buffer(xt.shape[0], xt.device)
    out = Q.topk_topp(xt, kt, pt, flags=Q.TruncFlags(**flags) if flags else None, kept_count=kept,
                      metrics=met, check=True)
    torch.cuda.synchronize()
    return out.float().cpu().numpy(), kept.cpu().numpy(), Q.ops.decode_metrics(met)


def assert_rows(x, got, kept, trip, label):
    want = G.masked_from_trip(x, trip)
    same = G.same_bits(got, want)
    bad = np.nonzero(~same.all(axis=1))[0]
    assert bad.size == 0, f"{label}: {bad.size} rows differ, first row {bad[0]}"
    assert np.array_equal(kept, trip[:, 2]), f"{label}: kept counts differ"


def test_kats(cuda_device):
    for row, k, p, keep in G.kats():
        out, kept, _ = run(row[None, :], [k], [p])
        want = np.where(keep, row, -np.inf).astype(np.float32)
        assert G.same_bits(out[0], want).all(), (row[:6], k, p, out[0][:6])
        assert kept[0] == keep.sum()


def test_signed_zero_bits_preserved(cuda_device):
    row = np.array([-0.0, 0.0, -0.0, 1.0, -0.0], dtype=np.float32)
    out, kept, _ = run(row[None, :], [3], [1.0])
    assert out[0].view(np.uint32).tolist()[:2] == [0x80000000, 0]
    assert np.isneginf(out[0][2]) and kept[0] == 3


def test_exhaustive_small_rows(cuda_device):
    z = G.exhaustive()
    vlen = z["vlen"]
    for v in np.unique(vlen):
        sel = np.nonzero(vlen == v)[0]
        x = np.ascontiguousarray(z["rows"][sel, :v])
        trip = np.stack([z["zb"][sel], z["cut"][sel], z["count"][sel]], axis=1).astype(np.int64)
        out, kept, _ = run(x, z["k"][sel], z["p"][sel])
        assert_rows(x, out, kept, trip, f"V={v}")


def test_acceptance_corpus_and_metrics(cuda_device):
    for key, x, k, p, trip, mets in G.corpus():
        out, kept, met = run(x, k, p)
        assert_rows(x, out, kept, trip, key)
        hit = np.array([m["trunc_hit"] for m in met])
        cnt = np.array([m["outlier_count"] for m in met])
        # reference RowMetrics parity: same sigma threshold -> same outlier counts and hit flags
        assert np.array_equal(cnt, mets["outlier_count"]), key
        assert np.array_equal(hit, mets["trunc_hit"].astype(bool)), key


@pytest.mark.parametrize("flags", [
    dict(search="binary"), dict(use_sigma_trunc=False), dict(force_fallback=True),
])
def test_ablation_flags_same_output(cuda_device, flags):
    for key, x, k, p, trip, _ in G.corpus():
        if x.shape[1] not in (8, 1000, 32768):
            continue
        out, kept, _ = run(x, k, p, **flags)
        assert_rows(x, out, kept, trip, f"{key} {flags}")


@pytest.mark.parametrize("run_id", ["C", "D", "E", "F", "H"])
@pytest.mark.parametrize("staged", [False, True])
def test_table3_ablations_vs_reference_pipeline(cuda_device, run_id, staged):
    """Table 3 runs C-H (cli.py:157-166) against the reference PIPELINE's own outputs under the same
    EngineConfig (tests/golden/ablation.npz): C / E (no duplicate handling) keep whole boundary
    clusters, D / F / H are exact."""
    for key, x, k, p, runs in G.ablation():
        out, kept, _ = run(x, k, p, staged=staged, **G.ABLATION_FLAGS[run_id])
        assert_rows(x, out, kept, runs[run_id], f"{key} run {run_id} staged={staged}")


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
def test_configs_full_size(cuda_device, name):
    x, k, p, dtype, trip, mets = G.config(name)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    out, kept, met = run(x, k, p, dtype=tdt)
    assert_rows(x, out, kept, trip, name)
    n = mets["outlier_count"].shape[0]
    assert np.array_equal(np.array([m["outlier_count"] for m in met[:n]]), mets["outlier_count"]), name
    assert np.array_equal(np.array([m["trunc_hit"] for m in met[:n]]), mets["trunc_hit"].astype(bool)), name


def test_bf16_output_bits(cuda_device):
    x, k, p, dtype, trip, _ = G.config("cfg3")
    xb = torch.from_numpy(to_bf16_bits(x[:4]).view(np.int16)).to("cuda").view(torch.bfloat16)
    out = Q.topk_topp(xb, torch.as_tensor(k[:4], device="cuda"), torch.as_tensor(p[:4], device="cuda"))
    ob = out.view(torch.int16).cpu().numpy().view(np.uint16)
    keep = np.stack([G.keep_from_trip(x[i], trip[i]) for i in range(4)])
    want = np.where(keep, to_bf16_bits(x[:4]), np.uint16(0xFF80))
    assert np.array_equal(ob, want)


def test_determinism_and_inplace(cuda_device):
    x, k, p, _, trip, _ = G.config("cfg2")
    xt = torch.from_numpy(x[:64]).cuda()
    kt, pt = torch.as_tensor(k[:64], device="cuda"), torch.as_tensor(p[:64], device="cuda")
    a = Q.topk_topp(xt, kt, pt)
    for _ in range(3):
        b = Q.topk_topp(xt, kt, pt)
        assert torch.equal(a.view(torch.int32), b.view(torch.int32))
    y = xt.clone()
    Q.topk_topp(y, kt, pt, inplace=True)
    assert torch.equal(a.view(torch.int32), y.view(torch.int32))


def test_random_ties_and_extremes(cuda_device):
    rng = np.random.default_rng(123)
    rows, ks, ps = [], [], []
    v = 3000
    for i in range(48):
        kind = i % 4
        if kind == 0:
            r = rng.integers(-3, 4, size=v).astype(np.float32)       # massive ties
        elif kind == 1:
            r = (rng.normal(size=v) * 40).astype(np.float32)          # wide spread, underflowing exp
        elif kind == 2:
            r = np.full(v, 2.5, np.float32)                            # all equal
        else:
            r = rng.normal(size=v).astype(np.float32) * 1e-30         # tiny logits
        rows.append(r)
        ks.append(int(rng.integers(1, v + 1)))
        ps.append(float(rng.choice([1e-12, 0.3, 0.9, 0.999999, 1.0])))
    x = np.stack(rows)
    out, kept, _ = run(x, ks, ps)
    for i in range(x.shape[0]):
        keep = oracle_keep_row(x[i], ks[i], ps[i])
        want = np.where(keep, x[i], -np.inf).astype(np.float32)
        assert G.same_bits(out[i], want).all(), (i, ks[i], ps[i])
        assert kept[i] == keep.sum()


def test_run_batch_dropin_numpy(cuda_device):
    batch = Q.synth_batch("gaussian", 16, 2048, seed=0)
    targets = Q.TruncTargets.uniform(16, 25, 0.9)
    out, rep = Q.run_batch(batch, targets, Q.EngineConfig())
    assert isinstance(out, np.ndarray) and out.dtype == np.float32
    want, _ = __import__("oracle.qrita_oracle", fromlist=["oracle_batch"]).oracle_batch(batch.values, 25, 0.9)
    assert G.same_bits(out, want).all()
    assert rep.hit_rate == 1.0 and len(rep.per_row) == 16
    with pytest.raises(ValueError, match="non-finite"):
        vals = np.zeros((2, 8), dtype=np.float32)
        vals[0, 0] = np.inf
        Q.run_batch(Q.LogitBatch(vals), Q.TruncTargets.uniform(2, 4, 1.0), Q.EngineConfig())


def test_device_side_nonfinite_status(cuda_device):
    x = torch.randn(3, 5000, device="cuda")
    x[1, 1234] = float("nan")
    with pytest.raises(ValueError, match="NaN logit at row 1, col 1234"):
        Q.topk_topp(x, 10, 0.9, check=True)
    with pytest.raises(ValueError, match="k out of range"):
        Q.topk_topp(torch.randn(2, 100, device="cuda"), torch.tensor([5, 101], device="cuda"), 0.5, check=True)


def test_pipeline_row_api(cuda_device):
    out = Q.truncate_topk(np.array([5, 5, 3, 5, 1], dtype=np.float32), 2)
    assert out.masked_row.tolist()[:2] == [5, 5] and out.kept_count == 2
    out = Q.truncate_topp(np.array([2, 1, 0], dtype=np.float32), 0.7)
    assert np.isneginf(out.masked_row[2]) and out.kept_count == 2
    row = np.array([3, 2, 1, 0], dtype=np.float32)
    res = Q.truncate_topk(row, 2, inplace=True)
    assert res.masked_row is row and np.isneginf(row[3])
    assert Q.truncate_topk(np.array([5, 5, 3, 5, 1], dtype=np.float32), 2, dup_handling=False).kept_count == 3
    with pytest.raises(ValueError):
        Q.truncate_topk(np.zeros(4, dtype=np.float32), 5)
    with pytest.raises(ValueError):
        Q.truncate_topp(np.zeros(4, dtype=np.float32), 1.5)


def test_verify_batch_with_exact_sort(cuda_device):
    batch = Q.synth_batch("quantized", 16, 512, seed=3, g=8)
    targets = Q.TruncTargets(np.arange(1, 17) * 7, np.linspace(0.3, 0.99, 16))
    assert Q.verify_batch(batch, targets, Q.EngineConfig()) == []


def test_outlier_spill_rows(cuda_device):
    """Rows whose sigma outliers exceed the fused kernel's shared-memory X (5632 entries) spill the rest
    to the row's HBM buffer and still take the bin-sort path; fp32 and bf16."""
    rng = np.random.default_rng(7)
    v = 262144
    x = rng.normal(size=(4, v)).astype(np.float32)
    ks, ps = [2000, 1500, 700, 1900], [0.9, 1.0, 0.8, 0.95]
    out, kept, met = run(x, ks, ps)
    assert max(m["outlier_count"] for m in met) > 5632
    assert all(m["full_row_path"] == 0 for m in met)
    for i in range(x.shape[0]):
        keep = oracle_keep_row(x[i], ks[i], ps[i])
        want = np.where(keep, x[i], -np.inf).astype(np.float32)
        assert G.same_bits(out[i], want).all(), i
        assert kept[i] == keep.sum()
    # kept-column lists of the same spill rows (index-only and beside the masked logits)
    xt = torch.from_numpy(x).cuda()
    kt = torch.tensor(ks, dtype=torch.int64, device="cuda")
    pt = torch.tensor(ps, dtype=torch.float64, device="cuda")
    for o in (None, torch.empty_like(xt)):
        kidx, kc = Q.topk_topp_indices(xt, kt, pt, out=o)
        got = _idx_sets(kidx.cpu().numpy(), kc.cpu().numpy())
        for i in range(x.shape[0]):
            assert np.array_equal(got[i], np.nonzero(oracle_keep_row(x[i], ks[i], ps[i]))[0]), i
    xb = to_bf16_bits(x[:2])
    xf = (xb.astype(np.uint32) << 16).view(np.float32)
    out, kept, _ = run(xf, ks[:2], ps[:2], dtype=torch.bfloat16)
    for i in range(2):
        keep = oracle_keep_row(xf[i], ks[i], ps[i])
        assert np.array_equal(~np.isneginf(out[i]), keep), i


def test_host_tensor_path(cuda_device):
    """Host tensors in, host tensors out: chunked transfers overlapped over the library's three
    streams (qrita_topk_topp_host); the chunks' status words land in one block, so errors still
    name the global row."""
    x, k, p, dtype, trip, _ = G.config("cfg2")
    n = 40  # 16 MB chunks of 32 rows -> 2 chunks
    xh = torch.from_numpy(np.ascontiguousarray(x[:n])).pin_memory()
    kept = torch.zeros(n, dtype=torch.int32, device="cuda")
    out = Q.topk_topp(xh, torch.from_numpy(k[:n]), torch.from_numpy(p[:n]), kept_count=kept)
    assert not out.is_cuda
    assert_rows(x[:n], out.numpy(), kept.cpu().numpy(), trip[:n], "host path")
    bad = xh.clone()
    bad[20, 5] = float("nan")
    with pytest.raises(ValueError, match="NaN logit at row 20, col 5"):
        Q.topk_topp(bad, torch.from_numpy(k[:n]), torch.from_numpy(p[:n]))


@pytest.mark.parametrize("dtype,pinned,chunk_rows", [(torch.float32, False, 7), (torch.bfloat16, True, 3),
                                                     (torch.float32, True, 1000)])
def test_host_path_chunking(cuda_device, dtype, pinned, chunk_rows):
    """qrita_topk_topp_host: pageable and pinned buffers, chunk sizes that do not divide B (and one
    larger than B), bf16, kept counts and metrics offset per chunk, precedence of row errors."""
    x, k, p, _, trip, _ = G.config("cfg2")
    n = 23
    xs = x[:n] if dtype == torch.float32 else torch.from_numpy(x[:n]).to(torch.bfloat16).float().numpy()
    xh = torch.from_numpy(np.ascontiguousarray(x[:n])).to(dtype)
    if pinned:
        xh = xh.pin_memory()
    kept = torch.zeros(n, dtype=torch.int32, device="cuda")
    met = Q.ops.metrics_buffer(n, "cuda")
    cb = chunk_rows * x.shape[1] * xh.element_size()
    out = Q.ops.topk_topp_host(xh, torch.from_numpy(k[:n]), torch.from_numpy(p[:n]), kept_count=kept,
                               metrics=met, chunk_bytes=cb)
    assert not out.is_cuda and out.dtype == dtype
    kc = kept.cpu().numpy()
    if dtype == torch.float32:
        assert_rows(x[:n], out.numpy(), kc, trip[:n], "host chunks")
    else:
        for r in range(n):
            ref = oracle_keep_row(xs[r], int(k[r]), float(p[r]))
            got = np.isfinite(out[r].float().numpy())
            assert np.array_equal(got, ref), f"bf16 host row {r}"
            assert kc[r] == ref.sum()
    rows = Q.ops.decode_metrics(met)
    assert [m["kept_count"] for m in rows] == list(kc)
    # k error in a late chunk, NaN in an earlier one: non-finite wins (core.py:120-140 order)
    bad = xh.clone()
    bad[4, 9] = float("nan")
    kb = torch.from_numpy(k[:n]).clone()
    kb[20] = 0
    with pytest.raises(ValueError, match="NaN logit at row 4, col 9"):
        Q.ops.topk_topp_host(bad, kb, torch.from_numpy(p[:n]), chunk_bytes=cb)
    with pytest.raises(ValueError, match="row 20"):
        Q.ops.topk_topp_host(xh, kb, torch.from_numpy(p[:n]), chunk_bytes=cb)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_random_sweep_fused_and_staged(cuda_device, seed):
    """Randomised shapes / distributions / targets through both pipelines (fused for 16-byte-aligned
    rows, staged otherwise and under QRITA_STAGED), fp32 and bf16, against the oracle."""
    rng = np.random.default_rng(1000 + seed)
    cases = []
    for v in (4096, 5000, 33000, 65536, 100003):
        for kind in ("normal", "ties", "wide", "spiky"):
            b = 6
            if kind == "normal":
                x = rng.normal(size=(b, v))
            elif kind == "ties":
                x = np.round(rng.normal(size=(b, v)) * 3) / 3
            elif kind == "wide":
                x = rng.normal(size=(b, v)) * 30
            else:  # a few huge logits on a gaussian bed (peaked distributions)
                x = rng.normal(size=(b, v))
                x[:, rng.integers(0, v, 5)] += 25.0
            k = rng.integers(1, min(v, 3000) + 1, b)
            k[0] = v  # top-p only
            p = rng.choice([0.3, 0.8, 0.95, 0.999, 1.0], b)
            cases.append((x.astype(np.float32), k, p))
    for x, k, p in cases:
        for dtype in (torch.float32, torch.bfloat16):
            xs = x if dtype == torch.float32 else \
                (to_bf16_bits(x).astype(np.uint32) << 16).view(np.float32)
            for staged in (False, True):
                out, kept, _ = run(xs, k, p, dtype=dtype, staged=staged)
                for i in range(xs.shape[0]):
                    keep = oracle_keep_row(xs[i], int(k[i]), float(p[i]))
                    assert np.array_equal(~np.isneginf(out[i]), keep), (xs.shape, dtype, staged, i, k[i], p[i])
                    assert kept[i] == keep.sum()
                    assert np.array_equal(out[i][keep].view(np.uint32), xs[i][keep].view(np.uint32))


def test_mixed_modes_many_rows_per_cta(cuda_device):
    """700 rows (several per persistent CTA) mixing pass-through, top-k, top-p-only, top-k+top-p,
    invalid k / p and non-finite rows: the ring's stage sequence runs across rows that take
    different resolve paths; valid rows stay exact and the status names the first bad row."""
    rng = np.random.default_rng(77)
    b, v = 700, 8192
    x = rng.normal(size=(b, v)).astype(np.float32)
    x[::7] = np.round(x[::7] * 2) / 2  # tie-heavy rows
    k = rng.integers(1, 2000, b)
    p = rng.choice([0.4, 0.9, 0.999, 1.0], b)
    mode = rng.integers(0, 4, b)
    k[mode == 0] = v; p[mode == 0] = 1.0   # pass-through
    k[mode == 1] = v                       # top-p only
    p[mode == 2] = 1.0                     # top-k only
    bad_k, bad_p, bad_nf = 101, 202, 303
    k[bad_k] = v + 5
    p[bad_p] = 0.0
    x[bad_nf, 4321] = np.inf
    xt = torch.from_numpy(x).cuda()
    kept = torch.zeros(b, dtype=torch.int32, device="cuda")
    out = Q.topk_topp(xt, torch.from_numpy(k).cuda(), torch.from_numpy(p).cuda(), kept_count=kept, check=False)
    torch.cuda.synchronize()
    got, kc = out.cpu().numpy(), kept.cpu().numpy()
    for i in range(b):
        if i in (bad_k, bad_p, bad_nf):
            continue
        keep = oracle_keep_row(x[i], int(k[i]), float(p[i]))
        want = np.where(keep, x[i], -np.inf).astype(np.float32)
        assert G.same_bits(got[i], want).all(), (i, k[i], p[i])
        assert kc[i] == keep.sum(), i
    with pytest.raises(ValueError, match="non-finite logit at row 303, col 4321"):
        Q.topk_topp(xt, torch.from_numpy(k).cuda(), torch.from_numpy(p).cuda(), check=True)


def test_row_passes_metric(cuda_device):
    """qrita_row_metrics.row_passes: the fused bin-sort path reads each logit once; full-row paths
    (forced fallback, top-p-only rows) report their extra passes."""
    x, k, p, dtype, trip, _ = G.config("cfg2")
    _, _, met = run(x[:32], k[:32], p[:32])
    assert all(m["row_passes"] == 1 for m in met)
    _, _, met = run(x[:4], k[:4], p[:4], force_fallback=True)
    assert all(m["row_passes"] > 1 for m in met)
    _, _, met = run(x[:4], np.full(4, x.shape[1]), np.full(4, 1.0))
    assert all(m["row_passes"] == 1 for m in met)


def test_capi_host_numpy_binding(cuda_device):
    """The INTEGRATION.md ctypes binding of qrita_topk_topp_host on plain (pageable) numpy arrays."""
    import ctypes
    from paper_2602_01518_b200 import _native as N
    lib = N.load()
    x, k, p, _, trip, _ = G.config("cfg2")
    n = 20
    xs = np.ascontiguousarray(x[:n]); out = np.empty_like(xs)
    kk = np.ascontiguousarray(k[:n], np.int64); pp = np.ascontiguousarray(p[:n], np.float64)
    B, V = xs.shape
    rows = 6
    nbytes = lib.qrita_host_scratch_bytes(B, V, 0, rows)
    scratch = torch.empty(nbytes + 256, dtype=torch.uint8, device="cuda")
    sp = (scratch.data_ptr() + 255) & ~255
    st = torch.cuda.current_stream().cuda_stream
    rc = lib.qrita_topk_topp_host(xs.ctypes.data, 0, B, V, kk.ctypes.data, pp.ctypes.data, out.ctypes.data,
                                  None, None, sp, nbytes, rows, 0, 4096, st)
    assert rc == N.OK
    row, col = ctypes.c_int(), ctypes.c_int()
    assert lib.qrita_get_status_host(sp, B, V, 0, rows, ctypes.byref(row), ctypes.byref(col), st) == N.OK
    kept = np.isfinite(out).sum(axis=1).astype(np.int32)
    assert_rows(xs, out, kept, trip[:n], "numpy host binding")
    # too-small scratch and bad arguments are rejected before any work is enqueued
    assert lib.qrita_topk_topp_host(xs.ctypes.data, 0, B, V, kk.ctypes.data, pp.ctypes.data, out.ctypes.data,
                                    None, None, sp, nbytes - 1, rows, 0, 4096, st) == N.EWORKSPACE
    assert lib.qrita_topk_topp_host(xs.ctypes.data, 0, B, V, kk.ctypes.data, pp.ctypes.data, out.ctypes.data,
                                    None, None, sp, nbytes, 0, 0, 4096, st) == N.EINVAL_ARG


def _idx_sets(kidx, kc):
    return [np.sort(kidx[r, :kc[r]]) for r in range(kidx.shape[0])]


@pytest.mark.parametrize("cfg", ["cfg2", "cfg3"])
def test_kept_indices_configs(cuda_device, cfg):
    """qrita_topk_topp_idx: index-only output (no masked logits) and indices beside the masked
    logits, against the golden kept sets (bin-sort rows of cfg2, distinct-value rows of cfg3)."""
    x, k, p, dtype, trip, _ = G.config(cfg)
    n = 64
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    xt = torch.from_numpy(np.ascontiguousarray(x[:n])).cuda().to(tdt)
    kt, pt = torch.from_numpy(k[:n]).cuda(), torch.from_numpy(p[:n]).cuda()
    want = [np.nonzero(G.keep_from_trip(x[r], trip[r]))[0] for r in range(n)]
    kidx, kc = Q.topk_topp_indices(xt, kt, pt)
    got = _idx_sets(kidx.cpu().numpy(), kc.cpu().numpy())
    for r in range(n):
        assert np.array_equal(got[r], want[r]), f"{cfg} index-only row {r}"
    out = torch.empty_like(xt)
    kidx, kc = Q.topk_topp_indices(xt, kt, pt, out=out)
    got = _idx_sets(kidx.cpu().numpy(), kc.cpu().numpy())
    o = out.float().cpu().numpy()
    for r in range(n):
        assert np.array_equal(got[r], want[r]), f"{cfg} indices beside logits row {r}"
        assert np.array_equal(np.nonzero(~np.isneginf(o[r]))[0], want[r])


def test_kept_indices_paths(cuda_device):
    """Every source of the kept list: pass-through rows, sorted candidates, X compaction (pivot
    search over the outliers), full-row compaction (fallback / top-p only / staged / unaligned V),
    fp32 and bf16, against the oracle."""
    rng = np.random.default_rng(77)
    for v in (4096, 5000, 40000):
        x = rng.normal(size=(8, v)).astype(np.float32)
        x[3] = np.round(x[3] * 3) / 3
        k = np.array([v, 50, 2000, 7, v, 300, 1, v], np.int64)
        p = np.array([1.0, 0.9, 0.8, 1.0, 0.95, 1.0, 0.5, 0.3])
        for dtype in (torch.float32, torch.bfloat16):
            xs = x if dtype == torch.float32 else (to_bf16_bits(x).astype(np.uint32) << 16).view(np.float32)
            want = [np.nonzero(oracle_keep_row(xs[r], int(k[r]), float(p[r])))[0] for r in range(8)]
            xt = torch.from_numpy(xs).cuda().to(dtype)
            for fl in (None, Q.TruncFlags(force_fallback=True), Q.TruncFlags(search="binary"), Q.TruncFlags(use_sigma_trunc=False),
                       Q.TruncFlags(staged=True)):
                kidx, kc = Q.topk_topp_indices(xt, torch.from_numpy(k).cuda(), torch.from_numpy(p).cuda(), flags=fl)
                got = _idx_sets(kidx.cpu().numpy(), kc.cpu().numpy())
                for r in range(8):
                    assert np.array_equal(got[r], want[r]), (v, dtype, fl, r, k[r], p[r])


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_host_sparse_download_pageable_out(cuda_device, dtype):
    """Pageable output + every row top-k (k <= 4096): only kept columns come back and the host builds
    the masked rows from its input copy — bit-identical to the dense download (QRITA_HOST_DENSE)
    and to the oracle; a top-p-only row in the batch switches the call to dense downloads."""
    import ctypes
    from paper_2602_01518_b200 import _native as N
    x, k, p, _, trip, _ = G.config("cfg2")
    n = 40
    xh = torch.from_numpy(np.ascontiguousarray(x[:n])).to(dtype)
    kh, ph = torch.from_numpy(k[:n]).clone(), torch.from_numpy(p[:n])
    out = torch.empty_like(xh)  # pageable
    lib = N.load()
    es = 4 if dtype == torch.float32 else 2
    sparse_bytes = lib.qrita_host_download_bytes(n, x.shape[1], 0 if es == 4 else 1, ctypes.c_void_p(kh.data_ptr()),
                                                 ctypes.c_void_p(xh.data_ptr()), ctypes.c_void_p(out.data_ptr()))
    assert 0 < sparse_bytes < n * x.shape[1] * es
    Q.ops.topk_topp_host(xh, kh, ph, out=out, chunk_bytes=9 * x.shape[1] * es)
    xs = xh.float().numpy()
    for r in range(n):
        ref = oracle_keep_row(xs[r], int(kh[r]), float(ph[r]))
        got = out[r].float().numpy()
        assert np.array_equal(np.isfinite(got), ref), r
        assert np.array_equal(got[ref], xs[r][ref]), r
    kh[7] = x.shape[1]                                # a top-p-only row: dense downloads
    assert lib.qrita_host_download_bytes(n, x.shape[1], 0 if es == 4 else 1, ctypes.c_void_p(kh.data_ptr()),
                                         ctypes.c_void_p(xh.data_ptr()),
                                         ctypes.c_void_p(out.data_ptr())) == n * x.shape[1] * es
    Q.ops.topk_topp_host(xh, kh, ph, out=out)
    ref = oracle_keep_row(xs[7], int(kh[7]), float(ph[7]))
    assert np.array_equal(np.isfinite(out[7].float().numpy()), ref)
