"""Step timing with and without CUDA-graph capture (isolates host launch overhead)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2602_01518_b200 as Q
import bench

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
x_np, k_np, p_np, dtype, desc, *_ = bench.workload(cfg)
tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
x = torch.from_numpy(x_np).cuda().to(tdt)
k = torch.from_numpy(k_np).cuda(); p = torch.from_numpy(p_np).cuda()
out = torch.empty_like(x)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream()
for _ in range(5):
    Q.topk_topp(x, k, p, out=out, check=True)
torch.cuda.synchronize()

def timeit(fn, n=30, do_flush=True):
    ts = []
    for _ in range(n):
        if do_flush:
            flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st); fn(); e1.record(st)
        ts.append((e0, e1))
    torch.cuda.synchronize()
    v = [a.elapsed_time(b) * 1e3 for a, b in ts]
    return statistics.median(v), min(v)

print(cfg, "eager      (median, min us):", timeit(lambda: Q.topk_topp(x, k, p, out=out, check=False)))
# delay the launch path: make sure the GPU is busy so the CPU runs ahead
g = torch.cuda.CUDAGraph()
s2 = torch.cuda.Stream()
s2.wait_stream(st)
with torch.cuda.stream(s2):
    Q.topk_topp(x, k, p, out=out, check=False)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s2):
        Q.topk_topp(x, k, p, out=out, check=False)
torch.cuda.synchronize()
print(cfg, "graph      (median, min us):", timeit(lambda: g.replay()))
print(cfg, "graph nofl (median, min us):", timeit(lambda: g.replay(), do_flush=False))
ref = Q.topk_topp(x, k, p, check=True)
g.replay(); torch.cuda.synchronize()
print("graph output identical:", torch.equal(ref.view(torch.int32), out.view(torch.int32)))
