import sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_2602_01518_b200.lmhead import lm_head_topk_topp
b, v, d = 256, 128256, 4096
h = torch.randn(b, d, device="cuda").to(torch.bfloat16)
w = (torch.randn(v, d, device="cuda") / d ** 0.5).to(torch.bfloat16)
rng = np.random.default_rng(2)
k = torch.from_numpy(rng.integers(1, 1025, b).astype(np.int64)).cuda()
p = torch.from_numpy(rng.uniform(0.5, 0.99, b)).cuda()
for _ in range(3):
    lm_head_topk_topp(h, w, k, p)
torch.cuda.synchronize()
