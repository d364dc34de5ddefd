"""PCIe pipeline without kernels: chunked H2D on one stream, D2H on another, D2H of chunk c after
H2D of chunk c (the host-buffer pipeline's dependency shape), vs chunk size; plus free-running."""
import sys, os, statistics
import torch
n = 131_334_144 // 4
xh = torch.empty(n, dtype=torch.float32).pin_memory(); oh = torch.empty_like(xh).pin_memory()
xd = torch.empty(n, device="cuda"); od = torch.empty(n, device="cuda")
up, down = torch.cuda.Stream(), torch.cuda.Stream()
cur = torch.cuda.current_stream()
def run(cb, dep):
    per = cb // 4
    spans = [(i, min(n, i + per)) for i in range(0, n, per)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cur); up.wait_stream(cur); down.wait_stream(cur)
    evs = []
    with torch.cuda.stream(up):
        for a, b in spans:
            xd[a:b].copy_(xh[a:b], non_blocking=True)
            ev = torch.cuda.Event(); ev.record(up); evs.append(ev)
    with torch.cuda.stream(down):
        for (a, b), ev in zip(spans, evs):
            if dep: down.wait_event(ev)
            oh[a:b].copy_(od[a:b], non_blocking=True)
    cur.wait_stream(up); cur.wait_stream(down); e1.record(cur)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)
for dep in (True, False):
    for cb in (1 << 20, 2 << 20, 4 << 20, 8 << 20, 16 << 20, 32 << 20):
        ts = [run(cb, dep) for _ in range(6)][2:]
        print(f"dep={dep} chunk {cb >> 20:3d} MB: {statistics.mean(ts):.3f} ms (min {min(ts):.3f})")
for d in ("h2d", "d2h"):
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        (xd.copy_(xh, non_blocking=True) if d == "h2d" else oh.copy_(od, non_blocking=True))
        e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print(d, "alone", round(min(ts), 3), "ms =", round(n * 4 / min(ts) / 1e6, 1), "GB/s")
