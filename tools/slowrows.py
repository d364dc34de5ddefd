"""Which rows are slow in the fused kernel (debug stamps) and what path they took (metrics)."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2602_01518_b200 as Q
from paper_2602_01518_b200 import _native as N
import bench
cfg = sys.argv[1]
x, k, p, dtype, desc, *_ = bench.workload(cfg)
xt = torch.from_numpy(x).cuda()
kt, pt = torch.from_numpy(k).cuda(), torch.from_numpy(p).cuda()
met = Q.ops.metrics_buffer(x.shape[0], xt.device)
fl = Q.TruncFlags(debug_timing=True)
st = torch.cuda.current_stream()
Q.topk_topp(xt, kt, pt, flags=fl, metrics=met)
ws = Q.ops.workspace_for(xt.device, st)
ptr, _ = ws.get(0, st)
B = x.shape[0]
buf = (ctypes.c_ulonglong * (16 * B))()
N.load().qrita_get_timing(ctypes.c_void_p(ptr), B, buf, ctypes.c_void_p(st.cuda_stream))
a = np.frombuffer(buf, dtype=np.uint64).reshape(B, 16).astype(np.int64)
m = Q.ops.decode_metrics(met)
res = (a[:, 9] - a[:, 2]) / 1e3
order = np.argsort(-res)[:8]
for r in order:
    print(r, f"resolve {res[r]:.1f} us", "k", k[r], "p", round(p[r], 3), m[r])
fr = [i for i in range(B) if m[i]["full_row_path"]]
print("full_row rows:", len(fr), fr[:20])
print("outliers max", max(mm["outlier_count"] for mm in m))
