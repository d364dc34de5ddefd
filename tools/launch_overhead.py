"""Event-timed launch overhead: empty kernels (0 / 115 KB shared memory, with / without a stack
frame) vs qrita_fused on tiny rows, each after a busy kernel so that host launch gaps are hidden."""
import sys, os, ctypes, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_01518_b200 as Q
lo = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "build", "exp", "lo.so"))
st = torch.cuda.current_stream()
SLEEP = int(os.environ.get('SLEEP', '1000000'))  # busy cycles before each timed launch (~0.5 ms)
def timeit(fn, n=40):
    ts = []
    for _ in range(n):
        torch.cuda._sleep(SLEEP)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); ts.append((a, b))
    torch.cuda.synchronize()
    v = [x.elapsed_time(y) * 1e3 for x, y in ts[5:]]
    return statistics.median(v), min(v)
S = 115 * 1024
cases = {
    "nothing": lambda: None,
    "empty 1x256": lambda: lo.lo_launch(0, 1, 0, ctypes.c_void_p(st.cuda_stream)),
    "smem115K 1": lambda: lo.lo_launch(1, 1, S, ctypes.c_void_p(st.cuda_stream)),
    "smem115K 256": lambda: lo.lo_launch(1, 256, S, ctypes.c_void_p(st.cuda_stream)),
    "stack+smem 1": lambda: lo.lo_launch(2, 1, S, ctypes.c_void_p(st.cuda_stream)),
    "stack+smem 256": lambda: lo.lo_launch(2, 256, S, ctypes.c_void_p(st.cuda_stream)),
}
for V in (1024, 32000):
    x = torch.randn(1, V, device="cuda"); o = torch.empty_like(x)
    kt = torch.full((1,), 50, dtype=torch.int64, device="cuda"); pt = torch.full((1,), 0.9, dtype=torch.float64, device="cuda")
    cases[f"qrita 1x{V}"] = (lambda x=x, o=o: Q.topk_topp(x, 50, 0.9, out=o, check=False))
    cases[f"qrita 1x{V} kt"] = (lambda x=x, o=o, kt=kt, pt=pt: Q.topk_topp(x, kt, pt, out=o, check=False))
x = torch.randn(256, 1024, device="cuda"); o = torch.empty_like(x)
cases["qrita 256x1024"] = lambda: Q.topk_topp(x, 50, 0.9, out=o, check=False)
for name, fn in cases.items():
    fn(); torch.cuda.synchronize()
import time
for name, fn in cases.items():
    torch.cuda._sleep(50000000); t0 = time.perf_counter()
    for _ in range(20): fn()
    print(f"host {name:16s} {(time.perf_counter() - t0) / 20 * 1e6:7.1f} us/call")
    torch.cuda.synchronize()
for rep in range(2):
    for name, fn in cases.items():
        m, mn = timeit(fn)
        print(f"{name:16s} median {m:6.2f} us  min {mn:6.2f}")
