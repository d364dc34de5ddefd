"""GPU-initiated PCIe traffic on pinned host memory (zero-copy): copy / read / write kernels over
the cfg2 matrix size, and scattered 4-byte writes (kept values) into a host row block."""
import os, sys, ctypes, statistics
import torch
zc = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "build", "exp", "zc.so"))
n = 256 * 128256
xh = torch.randn(n).pin_memory(); oh = torch.empty(n).pin_memory()
sink = torch.empty(4, device="cuda")
st = torch.cuda.current_stream()
def t(fn, reps=5):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return min(ts)
S = ctypes.c_void_p(st.cuda_stream)
ms = t(lambda: zc.zc_launch(0, ctypes.c_void_p(xh.data_ptr()), ctypes.c_void_p(oh.data_ptr()), n, S))
print(f"copy host->host via kernel: {ms:.3f} ms, {n*4/ms/1e6:.1f} GB/s each way"); assert torch.equal(xh, oh)
ms = t(lambda: zc.zc_launch(1, ctypes.c_void_p(xh.data_ptr()), ctypes.c_void_p(sink.data_ptr()), n, S))
print(f"read host via kernel: {ms:.3f} ms, {n*4/ms/1e6:.1f} GB/s")
ms = t(lambda: zc.zc_launch(2, ctypes.c_void_p(oh.data_ptr()), None, n, S))
print(f"write host via kernel: {ms:.3f} ms, {n*4/ms/1e6:.1f} GB/s")
for cnt in (256 * 512, 256 * 1024):
    idx = torch.randint(0, n, (cnt,), dtype=torch.int32, device="cuda")
    ms = t(lambda: zc.zc_launch(3, ctypes.c_void_p(oh.data_ptr()), ctypes.c_void_p(idx.data_ptr()), cnt, S))
    print(f"scatter {cnt} 4-byte writes to host: {ms:.3f} ms")
    idx, _ = torch.sort(idx)
    ms = t(lambda: zc.zc_launch(3, ctypes.c_void_p(oh.data_ptr()), ctypes.c_void_p(idx.data_ptr()), cnt, S))
    print(f"sorted scatter {cnt}: {ms:.3f} ms")
