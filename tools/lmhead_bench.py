"""LM-head fusion timing (B200): the tcgen05 GEMM alone, GEMM + topk_topp_indices (unfused), the fused
lm_head_topk_topp, and torch's bf16 matmul (cuBLAS) for scale.  L2 flushed before every timed call
(256 MB write + read-back), CUDA events on the current stream.
usage: python tools/lmhead_bench.py [B V d]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2602_01518_b200 as Q
from paper_2602_01518_b200.lmhead import lm_head_logits, lm_head_topk_topp

b, v, d = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (256, 128256, 4096)
torch.manual_seed(0)
h = torch.randn(b, d, device="cuda").to(torch.bfloat16)
w = (torch.randn(v, d, device="cuda") / d ** 0.5).to(torch.bfloat16)
rng = np.random.default_rng(2)
k = torch.from_numpy(rng.integers(1, 1025, b).astype(np.int64)).cuda()
p = torch.from_numpy(rng.uniform(0.5, 0.99, b)).cuda()
flush = torch.empty(64 << 20, device="cuda")
sink = torch.empty(1, device="cuda")
logits = torch.empty(b, v, device="cuda")


def timeit(fn, n=20, warm=3):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(n):
        flush.zero_()
        torch.sum(flush, dim=0, keepdim=True, out=sink)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        ts.append((e0, e1))
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(c) * 1e3 for a, c in ts)


res = {}
res["gemm (tcgen05, fp32 logits)"] = timeit(lambda: lm_head_logits(h, w, out=logits))
res["gemm + topk_topp_indices (unfused)"] = timeit(
    lambda: Q.topk_topp_indices(lm_head_logits(h, w, out=logits), k, p))
res["lm_head_topk_topp (fused)"] = timeit(lambda: lm_head_topk_topp(h, w, k, p))
res["torch bf16 matmul (cuBLAS, bf16 out)"] = timeit(lambda: h @ w.T)
wbytes = v * d * 2
flops = 2.0 * b * v * d
print(f"B={b} V={v} d={d}: weight {wbytes / 1e9:.2f} GB, {flops / 1e12:.2f} TFLOP")
for name, us in res.items():
    print(f"  {name:40s} {us:9.1f} us   {wbytes / us / 1e3:7.0f} GB/s of weight   {flops / us / 1e6:7.1f} TFLOP/s")
