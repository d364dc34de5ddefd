"""cfg1 (one row) latency after different preceding kernels: torch flush (small shared-memory
configuration) vs nothing vs another qrita_fused launch (same large shared-memory configuration)."""
import sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2602_01518_b200 as Q
import bench
x, k, p, dtype, desc, *_ = bench.workload("cfg1")
xt = torch.from_numpy(x).cuda(); kt, pt = torch.from_numpy(k).cuda(), torch.from_numpy(p).cuda(); out = torch.empty_like(xt)
fl = torch.empty(64 << 20, device="cuda"); sink = torch.empty(1, device="cuda")
tiny = torch.randn(1, 4096, device="cuda"); tout = torch.empty_like(tiny)
def torch_flush(): fl.zero_(); torch.sum(fl, dim=0, keepdim=True, out=sink)
def none(): pass
def sleep(): torch.cuda._sleep(200000)  # ~100 us busy kernel: keeps the queue full, L2 untouched
def qrita_pre(): torch_flush(); Q.topk_topp(tiny, 4096, 1.0, out=tout, check=False)
for name, pre in (("torch flush", torch_flush), ("sleep (warm L2)", sleep), ("flush + qrita", qrita_pre)) * 2:
    ts = []
    for i in range(40):
        pre()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); Q.topk_topp(xt, kt, pt, out=out, check=False); e1.record()
        ts.append((e0, e1))
    torch.cuda.synchronize()
    v = [a.elapsed_time(b) * 1e3 for a, b in ts[5:]]
    print(f"{name:14s}: median {statistics.median(v):5.1f} us  min {min(v):5.1f}")
