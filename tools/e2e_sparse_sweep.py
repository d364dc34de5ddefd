"""cfg2 end to end through Q.ops.topk_topp_host (pinned in / pinned out): dense downloads
(QRITA_HOST_DENSE=1) vs sparse (kept columns, host-built rows; the default here) over chunk sizes."""
import sys, os, statistics, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) < 2:
    for mode in ("dense", "sparse"):
        env = dict(os.environ)
        env["QRITA_HOST_DENSE" if mode == "dense" else "QRITA_HOST_SPARSE"] = "1"
        subprocess.run([sys.executable, __file__, mode], env=env)
    sys.exit(0)
import torch
import paper_2602_01518_b200 as Q
import bench
x_np, k_np, p_np, *_ = bench.workload("cfg2")
xh = torch.from_numpy(x_np).pin_memory(); oh = torch.empty_like(xh).pin_memory()
kh, ph = torch.from_numpy(k_np), torch.from_numpy(p_np)
st = torch.cuda.current_stream()
for cb in (2 << 20, 4 << 20, 8 << 20, 16 << 20):
    ts = []
    for i in range(8):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        Q.ops.topk_topp_host(xh, kh, ph, out=oh, chunk_bytes=cb)
        e1.record(st)
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    print(f"{sys.argv[1]:6s} chunk {cb >> 20:3d} MB: {statistics.mean(ts):.3f} ms (min {min(ts):.3f})", flush=True)
