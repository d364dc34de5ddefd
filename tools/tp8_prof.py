"""cfg5 through the TP protocol at world 8 (ranks as threads on one GPU: simulate_tp), for the
per-kernel durations of a TP=8 rank under ncu (the exchange is host-staged here)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2602_01518_b200.tp import simulate_tp
b, v = 128, 262144
x = torch.from_numpy(np.random.default_rng(5).normal(0, 1, (b, v)).astype(np.float32)).cuda()
r = np.random.default_rng(55)
k = torch.from_numpy(r.integers(1, 1025, b).astype(np.int64)).cuda()
p = torch.from_numpy(r.uniform(0.5, 0.99, b)).cuda()
for _ in range(2):
    simulate_tp(x, k, p, world=8)
torch.cuda.synchronize()
