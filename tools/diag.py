"""Diagnostics: run small cases on the GPU and print mismatches against the oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2602_01518_b200 as Q
from oracle.qrita_oracle import oracle_keep_row

def run(x, k, p, **fl):
    xt = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    kt = torch.as_tensor(np.asarray(k, np.int64), device="cuda"); pt = torch.as_tensor(np.asarray(p, np.float64), device="cuda")
    kept = torch.zeros(x.shape[0], dtype=torch.int32, device="cuda")
    met = Q.ops.metrics_buffer(x.shape[0], xt.device)
    out = Q.topk_topp(xt, kt, pt, kept_count=kept, metrics=met, flags=Q.TruncFlags(**fl) if fl else None)
    return out.cpu().numpy(), kept.cpu().numpy(), Q.ops.decode_metrics(met)

def check(name, x, k, p, maxshow=4, **fl):
    out, kept, met = run(x, k, p, **fl)
    nbad = 0
    for i in range(x.shape[0]):
        keep = oracle_keep_row(x[i], int(k[i]), float(p[i]))
        got = ~np.isneginf(out[i])
        if not np.array_equal(got, keep) or kept[i] != keep.sum():
            nbad += 1
            if nbad <= maxshow:
                print(f"  [{name}] row {i} V={x.shape[1]} k={k[i]} p={p[i]!r} want {keep.sum()} got {got.sum()} kept_count {kept[i]}")
                print(f"     met {met[i]}")
                if x.shape[1] <= 16:
                    print("     row", x[i].tolist(), "want", keep.astype(int).tolist(), "got", got.astype(int).tolist())
    print(f"{name}: {nbad}/{x.shape[0]} bad")

if len(sys.argv) > 1 and sys.argv[1] == "stats":
    pass
else:
  rng = np.random.default_rng(0)
  # 1. tiny top-p rows
  x = np.array([[2,1,0,0],[0,0,0,0],[9,0,0,0],[1,2,3,4]], np.float32)
  check("tiny-topp", x, [4]*4, [0.7,0.5,0.5,0.9])
  check("tiny-topk", x, [2]*4, [1.0]*4)
  check("tiny-comb", x, [3]*4, [0.9]*4)
  x = rng.normal(size=(16, 1000)).astype(np.float32)
  check("g1000-topp", x, [1000]*16, rng.uniform(0.1, 0.99, 16))
  check("g1000-topk", x, rng.integers(1, 1000, 16), [1.0]*16)
  check("g1000-comb", x, rng.integers(1, 1000, 16), rng.uniform(0.1, 0.99, 16))
  check("g1000-topp-nosigma", x, [1000]*16, rng.uniform(0.1, 0.99, 16), use_sigma_trunc=False)
  check("g1000-topk-nosigma", x, rng.integers(1, 1000, 16), [1.0]*16, use_sigma_trunc=False)
  x = rng.normal(size=(8, 40000)).astype(np.float32)
  check("g40000-topp", x, [40000]*8, rng.uniform(0.5, 0.99, 8))
  check("g40000-comb", x, rng.integers(1, 1024, 8), rng.uniform(0.5, 0.99, 8))
  check("g40000-comb-ff", x, rng.integers(1, 1024, 8), rng.uniform(0.5, 0.99, 8), force_fallback=True)
  xq = np.round(rng.normal(size=(8, 3000))*2).astype(np.float32)
  check("q3000-topk", xq, rng.integers(1, 3000, 8), [1.0]*8)
  check("q3000-topp", xq, [3000]*8, rng.uniform(0.1, 0.99, 8))
  # exhaustive-like for top-k V=5
  import itertools
  rows = np.array(list(itertools.product((0.,1.,2.), repeat=5)), np.float32)
  for kk in range(1, 6):
      check(f"exh5-k{kk}", rows, [kk]*len(rows), [1.0]*len(rows), maxshow=2)

if len(sys.argv) > 1 and sys.argv[1] == "stats":
    import bench
    for cfg in sys.argv[2:]:
        x, k, p, dtype, desc, *_ = bench.workload(cfg)
        tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
        xt = torch.from_numpy(x).cuda().to(tdt)
        met = Q.ops.metrics_buffer(x.shape[0], xt.device)
        Q.topk_topp(xt, torch.from_numpy(k).cuda(), torch.from_numpy(p).cuda(), metrics=met)
        m = Q.ops.decode_metrics(met)
        import statistics as st
        for f in ("trunc_hit", "outlier_count", "k_search_iters", "p_search_iters", "kept_count", "full_row_path"):
            vals = [r[f] for r in m]
            print(f"{cfg} {f}: mean {st.mean(vals):.2f} max {max(vals)}")

if len(sys.argv) > 1 and sys.argv[1] == "wtiming":
    import bench, ctypes
    from paper_2602_01518_b200 import _native as N
    for cfg in sys.argv[2:]:
        x, k, p, dtype, desc, *_ = bench.workload(cfg)
        xt = torch.from_numpy(x).cuda()
        kt, pt = torch.from_numpy(k).cuda(), torch.from_numpy(p).cuda()
        fl = Q.TruncFlags(debug_timing=True)
        for _ in range(3):
            Q.topk_topp(xt, kt, pt, flags=fl)
        torch.cuda.synchronize()
        st = torch.cuda.current_stream()
        ws = Q.ops.workspace_for(xt.device, st)
        ptr, _ = ws.get(0, st)
        B = x.shape[0]
        buf = (ctypes.c_ulonglong * (16 * B))()
        N.load().qrita_get_timing(ctypes.c_void_p(ptr), B, buf, ctypes.c_void_p(st.cuda_stream))
        a = np.frombuffer(buf, dtype=np.uint64).reshape(B, 16).astype(np.int64)
        t0 = a[:, 0]
        print(f"{cfg}: row completion spread {(t0.max()-t0.min())/1e3:.1f} us; last tail end {(a[:,9].max()-t0.min())/1e3:.1f} us")
        names = ["lock", "stats", "stage", "kbracket", "kpivot", "S+D+pi", "pbracket", "ppivot", "scatter"]
        prev = a[:, 0]
        for i, nm in enumerate(names, start=1):
            cur = a[:, i]
            ok = cur > 0
            d = np.where(ok, cur - prev, 0)
            print(f"   {nm:9s} mean {d[ok].mean()/1e3 if ok.any() else 0:8.2f} us  max {d.max()/1e3:8.2f}")
            prev = np.where(ok, cur, prev)

if len(sys.argv) > 1 and sys.argv[1] == "timing":
    import bench, ctypes
    from paper_2602_01518_b200 import _native as N
    for cfg in sys.argv[2:]:
        x, k, p, dtype, desc, *_ = bench.workload(cfg)
        tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
        xt = torch.from_numpy(x).cuda().to(tdt)
        kt, pt = torch.from_numpy(k).cuda(), torch.from_numpy(p).cuda()
        fl = Q.TruncFlags(debug_timing=True)
        for _ in range(3):
            Q.topk_topp(xt, kt, pt, flags=fl)
        torch.cuda.synchronize()
        st = torch.cuda.current_stream()
        ws = Q.ops.workspace_for(xt.device, st)
        ptr, _ = ws.get(0, st)
        B = x.shape[0]
        buf = (ctypes.c_ulonglong * (16 * B))()
        N.load().qrita_get_timing(ctypes.c_void_p(ptr), B, buf, ctypes.c_void_p(st.cuda_stream))
        a = np.frombuffer(buf, dtype=np.uint64).reshape(B, 16).astype(np.int64)
        t0 = a[:, 0]
        print(f"{cfg}: tail start spread {(t0.max()-t0.min())/1e3:.1f} us; total tail span {(a[:,9].max()-t0.min())/1e3:.1f} us")
        names = ["stats", "stageX", "ksearch", "kcut", "S+D", "Ml0", "psearch", "pcut", "output"]
        prev = a[:, 0]
        for i, nm in enumerate(names, start=1):
            cur = a[:, i]
            ok = cur > 0
            d = np.where(ok, cur - prev, 0)
            print(f"   {nm:8s} mean {d[ok].mean()/1e3 if ok.any() else 0:7.2f} us  max {d.max()/1e3:7.2f}")
            prev = np.where(ok, cur, prev)
        # bin-sort sub-phases (stamps 10-14 between stageX=2 and ksearch=3)
        sub = ["binscan", "scatter", "fixup", "expD", "piscan", "cross"]
        prev = a[:, 2]
        for j, nm in enumerate(sub):
            cur = a[:, 10 + j] if j < 5 else a[:, 3]
            ok = (cur > 0) & (prev > 0)
            d = np.where(ok, cur - prev, 0)
            print(f"     {nm:8s} mean {d[ok].mean()/1e3 if ok.any() else 0:7.2f} us  max {d.max()/1e3:7.2f}")
            prev = np.where(cur > 0, cur, prev)

if len(sys.argv) > 1 and sys.argv[1] == "ftiming":
    # fused kernel: per-row phases (0 row start, 1 plan, 2 streamed, 9 end) and the CTA timeline
    import bench, ctypes
    from paper_2602_01518_b200 import _native as N
    for cfg in sys.argv[2:]:
        x, k, p, dtype, desc, *_ = bench.workload(cfg)
        tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
        xt = torch.from_numpy(x).cuda().to(tdt)
        kt, pt = torch.from_numpy(k).cuda(), torch.from_numpy(p).cuda()
        fl = Q.TruncFlags(debug_timing=True)
        # IDX=1: index-only output (topk_topp_indices, no masked logits)
        call = (lambda *a, **kw: Q.topk_topp_indices(*a, **kw)) if os.environ.get("IDX") else Q.topk_topp
        st = torch.cuda.current_stream()
        ws = Q.ops.workspace_for(xt.device, st)
        for _ in range(3):
            call(xt, kt, pt, flags=fl)
        ptr, _ = ws.get(0, st)
        B = x.shape[0]
        ws.buf.zero_()
        if os.environ.get("FLUSH"):  # evict the kernel's code and data from L2 first (serving-like)
            fl_buf = torch.empty(64 << 20, device="cuda"); fl_buf.zero_(); fl_buf.sum()
        call(xt, kt, pt, flags=fl)
        buf = (ctypes.c_ulonglong * (16 * B))()
        N.load().qrita_get_timing(ctypes.c_void_p(ptr), B, buf, ctypes.c_void_p(st.cuda_stream))
        a = np.frombuffer(buf, dtype=np.uint64).reshape(B, 16).astype(np.int64)
        t0 = a[:, 0].min()
        end = np.where(a[:, 9] > 0, a[:, 9], a[:, 2])
        print(f"{cfg}: B={B} flush={bool(os.environ.get('FLUSH'))} start spread {(a[:,0].max()-t0)/1e3:.1f} us, last end {(end.max()-t0)/1e3:.1f} us")
        for nm, i, j in (("plan", 0, 1), ("stream", 1, 2), ("resolve", 2, 9)):
            ok = (a[:, i] > 0) & (a[:, j] > 0)
            d = (a[ok, j] - a[ok, i]) / 1e3
            if ok.any():
                print(f"   {nm:8s} mean {d.mean():7.2f} us  min {d.min():7.2f}  max {d.max():7.2f}")
        sub = ((("binscan", 2, 10), ("scatter", 10, 11), ("fixup+e", 11, 12), ("D", 12, 13),
                ("piscan", 13, 14), ("cross", 14, 3), ("output", 3, 9)) if cfg != "cfg3" else
               (("count", 2, 10), ("sort", 10, 11), ("masses", 11, 12), ("select", 12, 13), ("output", 13, 9)))
        for nm, i, j in sub:
            ok = (a[:, i] > 0) & (a[:, j] > 0)
            d = (a[ok, j] - a[ok, i]) / 1e3
            if ok.any():
                print(f"     {nm:8s} mean {d.mean():7.2f} us  max {d.max():7.2f}")
        q = np.percentile((a[:, 0] - t0) / 1e3, [0, 25, 50, 75, 100])
        print("   row start percentiles", np.round(q, 1))
        q = np.percentile((end - t0) / 1e3, [0, 25, 50, 75, 100])
        print("   row end percentiles  ", np.round(q, 1))

if len(sys.argv) > 1 and sys.argv[1] == "smid":
    # fused kernel: stream time of rows on SMs that host one vs two rows
    import bench, ctypes
    from paper_2602_01518_b200 import _native as N
    cfg = sys.argv[2] if len(sys.argv) > 2 else "cfg2"
    x, k, p, dtype, desc, *_ = bench.workload(cfg)
    xt = torch.from_numpy(x).cuda()
    kt, pt = torch.from_numpy(k).cuda(), torch.from_numpy(p).cuda()
    fl = Q.TruncFlags(debug_timing=True)
    st = torch.cuda.current_stream()
    for _ in range(3):
        Q.topk_topp(xt, kt, pt, flags=fl)
    ws = Q.ops.workspace_for(xt.device, st)
    ptr, _ = ws.get(0, st)
    B = x.shape[0]
    for rep in range(3):
        ws.buf.zero_()
        Q.topk_topp(xt, kt, pt, flags=fl)
        buf = (ctypes.c_ulonglong * (16 * B))()
        N.load().qrita_get_timing(ctypes.c_void_p(ptr), B, buf, ctypes.c_void_p(st.cuda_stream))
        a = np.frombuffer(buf, dtype=np.uint64).reshape(B, 16).astype(np.int64)
        sm = a[:, 15]
        cnt = np.bincount(sm, minlength=148)
        per = cnt[sm]
        stream = (a[:, 2] - a[:, 1]) / 1e3
        end = (a[:, 9] - a[:, 0].min()) / 1e3
        for n in (1, 2):
            sel = per == n
            if sel.any():
                print(f"rep{rep} rows on {n}-row SMs: {sel.sum():3d}  stream mean {stream[sel].mean():6.2f} max {stream[sel].max():6.2f}  end mean {end[sel].mean():6.2f} max {end[sel].max():6.2f}")

if len(sys.argv) > 1 and sys.argv[1] == "smidmap":
    # per-SM stream time over several runs: are slow rows tied to particular SMs?
    import bench, ctypes
    from paper_2602_01518_b200 import _native as N
    x, k, p, dtype, desc, *_ = bench.workload("cfg2")
    xt = torch.from_numpy(x).cuda()
    kt, pt = torch.from_numpy(k).cuda(), torch.from_numpy(p).cuda()
    fl = Q.TruncFlags(debug_timing=True)
    st = torch.cuda.current_stream()
    for _ in range(3):
        Q.topk_topp(xt, kt, pt, flags=fl)
    ws = Q.ops.workspace_for(xt.device, st)
    ptr, _ = ws.get(0, st)
    B = x.shape[0]
    acc = np.zeros(148); n = np.zeros(148)
    for rep in range(8):
        ws.buf.zero_()
        Q.topk_topp(xt, kt, pt, flags=fl)
        buf = (ctypes.c_ulonglong * (16 * B))()
        N.load().qrita_get_timing(ctypes.c_void_p(ptr), B, buf, ctypes.c_void_p(st.cuda_stream))
        a = np.frombuffer(buf, dtype=np.uint64).reshape(B, 16).astype(np.int64)
        sm = a[:, 15]
        stream = (a[:, 2] - a[:, 1]) / 1e3
        np.add.at(acc, sm, stream); np.add.at(n, sm, 1)
    mean = acc / np.maximum(n, 1)
    order = np.argsort(-mean)
    print("slowest SMs (smid: mean stream us, rows):", [(int(i), round(mean[i], 1), int(n[i] / 8)) for i in order[:12]])
    print("fastest SMs:", [(int(i), round(mean[i], 1), int(n[i] / 8)) for i in order[-8:]])
    two = n / 8 == 2
    print("2-row SMs: smid<74 mean", round(mean[two & (np.arange(148) < 74)].mean(), 2), " smid>=74 mean", round(mean[two & (np.arange(148) >= 74)].mean(), 2))
    print("per-SM std over 2-row SMs", round(mean[two].std(), 2))

if len(sys.argv) > 1 and sys.argv[1] == "t16timing":
    # qrita_topp16 (bf16 top-p-only rows): per-row phase stamps of the cluster's CTA 0
    import bench, ctypes
    from paper_2602_01518_b200 import _native as N
    x, k, p, dtype, desc, *_ = bench.workload("cfg3")
    xt = torch.from_numpy(x).cuda().to(torch.bfloat16)
    kt, pt = torch.from_numpy(k).cuda(), torch.from_numpy(p).cuda()
    fl = Q.TruncFlags(debug_timing=True)
    st = torch.cuda.current_stream()
    ws = Q.ops.workspace_for(xt.device, st)
    for _ in range(3):
        Q.topk_topp(xt, kt, pt, flags=fl)
    ptr, _ = ws.get(0, st)
    B = x.shape[0]
    buf = (ctypes.c_ulonglong * (16 * B))()
    N.load().qrita_get_timing(ctypes.c_void_p(ptr), B, buf, ctypes.c_void_p(st.cuda_stream))
    a = np.frombuffer(buf, dtype=np.uint64).reshape(B, 16).astype(np.int64)
    t0 = a[:, 0].min()
    print(f"cfg3 topp16: start spread {(a[:,0].max()-t0)/1e3:.1f} us, last end {(a[:,6].max()-t0)/1e3:.1f} us")
    for nm, i, j in (("count", 0, 1), ("sync1", 1, 2), ("merge+D", 2, 3), ("mass", 3, 7), ("suffix", 7, 8),
                     ("sync3", 8, 9), ("xfind", 9, 10), ("xwarp+s4", 10, 4), ("kept", 4, 5),
                     ("output", 5, 6), ("out(cta1)", 12, 13)):
        d = (a[:, j] - a[:, i]) / 1e3
        print(f"   {nm:10s} mean {d.mean():7.2f} us  min {d.min():7.2f}  max {d.max():7.2f}")
