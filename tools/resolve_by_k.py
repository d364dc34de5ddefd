import os, sys, ctypes
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
import paper_2602_01518_b200 as Q
from paper_2602_01518_b200 import _native as N
x, k, p, *_ = bench.workload("cfg2")
xt = torch.from_numpy(x).cuda(); kt = torch.from_numpy(k).cuda(); pt = torch.from_numpy(p).cuda()
fl = Q.TruncFlags(debug_timing=True)
st = torch.cuda.current_stream()
for _ in range(3): Q.topk_topp(xt, kt, pt, flags=fl)
ws = Q.ops.workspace_for(xt.device, st); ptr, _ = ws.get(0, st)
B = x.shape[0]
flush = torch.empty(64 << 20, device="cuda")
ws.buf.zero_(); flush.zero_(); flush.sum()
Q.topk_topp(xt, kt, pt, flags=fl)
buf = (ctypes.c_ulonglong * (16 * B))()
N.load().qrita_get_timing(ctypes.c_void_p(ptr), B, buf, ctypes.c_void_p(st.cuda_stream))
a = np.frombuffer(buf, dtype=np.uint64).reshape(B, 16).astype(np.int64)
o = np.argsort(k)
names = (("binscan", 2, 10), ("scatter", 10, 11), ("fixup+e", 11, 12), ("D", 12, 13), ("piscan", 13, 14), ("cross", 14, 3), ("output", 3, 9), ("total", 2, 9))
for q in range(4):
    sl = o[q * 64:(q + 1) * 64]
    parts = []
    for nm, i, j in names:
        ok = (a[sl, i] > 0) & (a[sl, j] > 0)
        d = (a[sl][ok, j] - a[sl][ok, i]) / 1e3
        parts.append(f"{nm} {d.mean():.2f}" if ok.any() else f"{nm} -")
    print(f"k {k[sl].min()}..{k[sl].max()}: " + "  ".join(parts))
