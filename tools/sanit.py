import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2602_01518_b200 as Q
B, V = int(sys.argv[1]), int(sys.argv[2])
r = np.random.default_rng(4)
x = torch.from_numpy(r.normal(0, 1, (B, V)).astype(np.float32)).cuda()
k = torch.from_numpy(r.integers(1, 1025, B).astype(np.int64)).cuda()
p = torch.from_numpy(r.uniform(0.5, 0.99, B)).cuda()
o = Q.topk_topp(x, k, p)
torch.cuda.synchronize()
print("ok", B, V, int((~torch.isinf(o)).sum()))
