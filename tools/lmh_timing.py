"""Per-tile epilogue phases of the fused LM-head GEMM (QRITA_LMH_TIMING=1): wait for the
accumulator, phase A (logits + per-row stats), B + C (reservation, outlier writes)."""
import os, sys, ctypes
os.environ["QRITA_LMH_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2602_01518_b200 import _native as N
from paper_2602_01518_b200.lmhead import lm_head_topk_topp
b, v, d = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (256, 128256, 4096)
h = torch.randn(b, d, device="cuda").to(torch.bfloat16)
w = (torch.randn(v, d, device="cuda") / d ** 0.5).to(torch.bfloat16)
k = torch.randint(1, 1025, (b,), device="cuda"); p = torch.rand(b, device="cuda", dtype=torch.float64) * 0.49 + 0.5
for _ in range(3):
    lm_head_topk_topp(h, w, k, p)
torch.cuda.synchronize()
lib = N.load()
lib.qrita_lmhead_timing.argtypes = [ctypes.c_void_p, ctypes.c_int]
n = 148 * 8 * 4
buf = (ctypes.c_ulonglong * n)()
assert lib.qrita_lmhead_timing(buf, n) == 0
a = np.frombuffer(buf, dtype=np.uint64).reshape(148, 8, 4).astype(np.int64)
t0 = a[:, 7, 0][a[:, 7, 0] > 0].min()
e = a[:, 7] - t0
print(f"epilogue entry -> tile-0 sample/acc {e[:,1].mean()/1e3:.1f} (max {e[:,1].max()/1e3:.1f}) -> own plans "
      f"{e[:,2].mean()/1e3:.1f} (max {e[:,2].max()/1e3:.1f}) us")
f = a[:, 6] - t0
print(f"samples complete {f[:,1].mean()/1e3:.1f} (max {f[:,1].max()/1e3:.1f})  plan_begin {((f[:,2]-f[:,1]).mean())/1e3:.2f}"
      f"  plan_sample {((f[:,3]-f[:,2]).mean())/1e3:.2f} us")
for i in range(6):
    ok = a[:, i, 0] > 0
    if not ok.any():
        break
    s = a[ok, i] - t0
    print(f"tile {i}: epi start {s[:,0].mean()/1e3:7.1f}  acc ready {s[:,1].mean()/1e3:7.1f} (max {s[:,1].max()/1e3:7.1f})"
          f"  A {((s[:,2]-s[:,1]).mean())/1e3:5.1f}  B+C {((s[:,3]-s[:,2]).mean())/1e3:5.1f} us  n={ok.sum()}")
