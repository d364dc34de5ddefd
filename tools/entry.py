import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2602_01518_b200 as Q
from paper_2602_01518_b200 import _native as N
import bench
for cfg in ("cfg1", "cfg2"):
    x, k, p, dtype, desc = bench.workload(cfg)
    xt = torch.from_numpy(x).cuda(); kt, pt = torch.from_numpy(k).cuda(), torch.from_numpy(p).cuda()
    fl = Q.TruncFlags(debug_timing=True); st = torch.cuda.current_stream()
    flush = torch.empty(64 << 20, device="cuda")
    for _ in range(3): Q.topk_topp(xt, kt, pt, flags=fl)
    ws = Q.ops.workspace_for(xt.device, st); ptr, _ = ws.get(0, st); B = x.shape[0]
    for rep in range(3):
        flush.zero_(); flush.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); Q.topk_topp(xt, kt, pt, flags=fl, check=False); e1.record(); torch.cuda.synchronize()
        buf = (ctypes.c_ulonglong * (16 * B))()
        N.load().qrita_get_timing(ctypes.c_void_p(ptr), B, buf, ctypes.c_void_p(st.cuda_stream))
        a = np.frombuffer(buf, dtype=np.uint64).reshape(B, 16).astype(np.int64)
        ent = a[:, 15]; t0 = ent.min()
        print(cfg, f"event {e0.elapsed_time(e1)*1e3:.1f} us | entry spread {(ent.max()-t0)/1e3:.2f} | entry->row start {(a[:,0]-ent).mean()/1e3:.2f} | entry->end max {(a[:,9].max()-t0)/1e3:.1f} | plan {(a[:,1]-a[:,0]).mean()/1e3:.2f} stream {(a[:,2]-a[:,1]).mean()/1e3:.2f} resolve {(a[:,9]-a[:,2]).mean()/1e3:.2f}")
