"""Which rows of cfg2 land on SMs that host one row (vs two), run to run, and how the resolve time
depends on k: the basis for the row order of the fused kernel."""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_2602_01518_b200 as Q
from paper_2602_01518_b200 import _native as N
x, k, p, *_ = bench.workload("cfg2")
xt = torch.from_numpy(x).cuda(); kt = torch.from_numpy(k).cuda(); pt = torch.from_numpy(p).cuda()
fl = Q.TruncFlags(debug_timing=True)
st = torch.cuda.current_stream()
for _ in range(3):
    Q.topk_topp(xt, kt, pt, flags=fl)
ws = Q.ops.workspace_for(xt.device, st)
ptr, _ = ws.get(0, st)
B = x.shape[0]
flush = torch.empty(64 << 20, device="cuda")
singles = []
for rep in range(4):
    ws.buf.zero_(); flush.zero_(); flush.sum()
    Q.topk_topp(xt, kt, pt, flags=fl)
    buf = (ctypes.c_ulonglong * (16 * B))()
    N.load().qrita_get_timing(ctypes.c_void_p(ptr), B, buf, ctypes.c_void_p(st.cuda_stream))
    a = np.frombuffer(buf, dtype=np.uint64).reshape(B, 16).astype(np.int64)
    sm = a[:, 15]
    per = np.bincount(sm, minlength=148)[sm]
    one = np.nonzero(per == 1)[0]
    singles.append(set(one.tolist()))
    print(f"rep{rep}: single-row SM rows {one.min()}..{one.max()} (n={len(one)}), smid of row 0..3: {sm[:4]}, row 148: {sm[148]}")
    res = (a[:, 9] - a[:, 2]) / 1e3
    if rep == 0:
        o = np.argsort(k)
        for q in range(4):
            sl = o[q * 64:(q + 1) * 64]
            print(f"   k quartile {q}: k {k[sl].min()}..{k[sl].max()}  resolve mean {res[sl].mean():.2f} max {res[sl].max():.2f}")
print("same single-row set every run:", all(s == singles[0] for s in singles))
