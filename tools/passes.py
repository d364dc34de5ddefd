import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2602_01518_b200 as Q
import bench
for cfg, fl in (("cfg2", None), ("cfg4", None), ("cfg3", None), ("cfg1", None), ("cfg2", Q.TruncFlags(force_fallback=True)), ("cfg2", Q.TruncFlags(use_sigma_trunc=False))):
    x, k, p, dtype, desc, *_ = bench.workload(cfg)
    n = min(x.shape[0], 64)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    xt = torch.from_numpy(x[:n]).cuda().to(tdt)
    met = Q.ops.metrics_buffer(n, xt.device)
    Q.topk_topp(xt, torch.from_numpy(k[:n]).cuda(), torch.from_numpy(p[:n]).cuda(), flags=fl, metrics=met)
    rp = [m["row_passes"] for m in Q.ops.decode_metrics(met)]
    print(cfg, "force_fb" if fl and fl.force_fallback else ("no_sigma" if fl else ""), "mean", round(sum(rp)/len(rp), 2), "min", min(rp), "max", max(rp))
