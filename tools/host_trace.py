"""Per-chunk timeline of qrita_topk_topp_host (QRITA_HOST_TRACE=1) on cfg2 for a few chunk sizes."""
import sys, os
os.environ["QRITA_HOST_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_01518_b200 as Q
import bench
x_np, k_np, p_np, dtype, desc, *_ = bench.workload("cfg2")
xh = torch.from_numpy(x_np).pin_memory(); oh = torch.empty_like(xh).pin_memory()
kh, ph = torch.from_numpy(k_np), torch.from_numpy(p_np)
for cb in [int(a) << 20 for a in (sys.argv[1:] or ["4", "16"])]:
    for i in range(3):
        print(f"--- chunk {cb >> 20} MB, call {i}", file=sys.stderr, flush=True)
        Q.ops.topk_topp_host(xh, kh, ph, out=oh, chunk_bytes=cb)
