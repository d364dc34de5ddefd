"""Does the L2-flush kernel's shared-memory configuration change the next qrita_fused step?"""
import sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2602_01518_b200 as Q
import bench
x, k, p, dtype, desc, *_ = bench.workload("cfg2")
xt = torch.from_numpy(x).cuda(); kt, pt = torch.from_numpy(k).cuda(), torch.from_numpy(p).cuda()
out = torch.empty_like(xt)
fl = torch.empty(64 << 20, device="cuda"); sink = torch.empty(1, device="cuda")
big = torch.randn(256, 262144, device="cuda"); bigo = torch.empty_like(big)
kb = torch.full((256,), 262144, dtype=torch.int64, device="cuda"); pb = torch.ones(256, dtype=torch.float64, device="cuda")
def torch_flush():
    fl.zero_(); torch.sum(fl, dim=0, keepdim=True, out=sink)
def qrita_flush():  # pass-through rows through the fused kernel: 256 MB read + 256 MB written
    Q.topk_topp(big, kb, pb, out=bigo, check=False)
for name, flush in (("torch", torch_flush), ("qrita", qrita_flush), ("torch", torch_flush), ("qrita", qrita_flush)):
    for _ in range(3):
        flush(); Q.topk_topp(xt, kt, pt, out=out, check=False)
    ts = []
    for _ in range(30):
        flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); Q.topk_topp(xt, kt, pt, out=out, check=False); e1.record()
        ts.append((e0, e1))
    torch.cuda.synchronize()
    v = [a.elapsed_time(b) * 1e3 for a, b in ts]
    print(f"flush={name}: median {statistics.median(v):.1f} us  min {min(v):.1f}")
