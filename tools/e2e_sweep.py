"""e2e (host tensors through Q.topk_topp) vs chunk size and stream count, cfg2."""
import sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2602_01518_b200 as Q
import bench
x_np, k_np, p_np, dtype, desc, *_ = bench.workload("cfg2")
xh = torch.from_numpy(x_np).pin_memory(); oh = torch.empty_like(xh).pin_memory()
kh, ph = torch.from_numpy(k_np), torch.from_numpy(p_np)
st = torch.cuda.current_stream()
for cb in (8 << 20, 16 << 20, 32 << 20):
  for ramp in ("1", "0"):
    os.environ["QRITA_HOST_RAMP"] = ramp
    for ns in (3,):
        ts = []
        for i in range(6):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            Q.ops.topk_topp_host(xh, kh, ph, out=oh, chunk_bytes=cb)
            e1.record(st)
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1))
        print(f"chunk {cb >> 20:3d} MB ramp {ramp}: {statistics.mean(ts):.3f} ms (min {min(ts):.3f})")
