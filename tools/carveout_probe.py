"""Does the SM shared-memory carveout switch cost the fused kernel launch time?  cfg2 timed after the
usual L2 flush (torch kernels, default carveout) vs after the flush plus a tiny call of a max-smem
kernel (qrita_topp16 on one bf16 row), CUDA events around the cfg2 call only."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2602_01518_b200 as Q
x, k, p, *_ = bench.workload("cfg2")
xt = torch.from_numpy(x).cuda(); kt = torch.from_numpy(k).cuda(); pt = torch.from_numpy(p).cuda()
out = torch.empty_like(xt)
tiny = torch.randn(1, 8192, device="cuda").to(torch.bfloat16)
tk = torch.tensor([8192], device="cuda"); tp = torch.tensor([0.9], dtype=torch.float64, device="cuda")
flush = torch.empty(64 << 20, device="cuda"); sink = torch.empty(1, device="cuda")
def t(pre, n=40):
    for _ in range(5): pre(); Q.topk_topp(xt, kt, pt, out=out)
    ev = []
    for _ in range(n):
        flush.zero_(); torch.sum(flush, dim=0, keepdim=True, out=sink); pre()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); Q.topk_topp(xt, kt, pt, out=out); b.record(); ev.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) * 1e3 for a, b in ev)
print("after torch flush only   %.1f us" % t(lambda: None))
print("after flush + max-smem   %.1f us" % t(lambda: Q.topk_topp(tiny, tk, tp)))
print("after flush only (again) %.1f us" % t(lambda: None))
