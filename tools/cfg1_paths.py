import sys, os, statistics
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_2602_01518_b200 as Q
import bench
x, k, p, *_ = bench.workload("cfg1")
xt = torch.from_numpy(x).cuda(); kt = torch.from_numpy(k).cuda(); pt = torch.from_numpy(p).cuda()
out = torch.empty_like(xt)
flush = torch.empty(64 << 20, device="cuda"); sink = torch.empty(1, device="cuda")
def t(fn, n=50):
    for _ in range(5): fn()
    ev = []
    for _ in range(n):
        flush.zero_(); torch.sum(flush, dim=0, keepdim=True, out=sink)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); ev.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) * 1e3 for a, b in ev)
print("fused", t(lambda: Q.topk_topp(xt, kt, pt, out=out)))
print("staged", t(lambda: Q.topk_topp(xt, kt, pt, out=out, flags=Q.TruncFlags(staged=True))))
print("idx fused", t(lambda: Q.topk_topp_indices(xt, kt, pt)))
