"""e2e host-buffer variants on cfg2: pinned / pageable input x pinned / pageable output, and run_batch."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_01518_b200 as Q  # noqa: E402

x = np.random.default_rng(1).normal(0.0, 1.0, (256, 128256)).astype(np.float32)
r = np.random.default_rng(42)
k = torch.from_numpy(r.integers(1, 1025, 256).astype(np.int64))
p = torch.from_numpy(r.uniform(0.5, 0.99, 256))


def t(fn, n=8):
    fn()
    fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return 1e3 * float(np.median(ts))


xp = torch.from_numpy(x)
xpin = xp.pin_memory()
opin = torch.empty_like(xpin).pin_memory()
opag = torch.empty_like(xp)
for name, xi, oi in (("pinned->pinned", xpin, opin), ("pageable->pinned", xp, opin),
                     ("pinned->pageable", xpin, opag), ("pageable->pageable", xp, opag)):
    print(f"{name:22s} {t(lambda: Q.topk_topp(xi, k, p, out=oi)):.2f} ms")
print(f"{'fresh numpy out':22s} {t(lambda: Q.topk_topp(xp, k, p, out=torch.from_numpy(np.empty_like(x)))):.2f} ms")
b, tg, cfg = Q.LogitBatch(x), Q.TruncTargets(k.numpy(), p.numpy()), Q.EngineConfig()
print(f"{'run_batch':22s} {t(lambda: Q.run_batch(b, tg, cfg)):.2f} ms")
for th in (4, 8):
    pass
