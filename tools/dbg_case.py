import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2602_01518_b200 as Q
from oracle.qrita_oracle import oracle_keep_row
from oracle.synth import to_bf16_bits
rng = np.random.default_rng(1000)
for v in (100003, 100000, 5001, 5000):
    x = rng.normal(size=(2, v)).astype(np.float32)
    xs = (to_bf16_bits(x).astype(np.uint32) << 16).view(np.float32)
    for dt in (torch.bfloat16, torch.float32):
        for staged in (False, True):
            xt = torch.from_numpy(xs).cuda().to(dt)
            met = Q.ops.metrics_buffer(2, xt.device)
            kept = torch.zeros(2, dtype=torch.int32, device="cuda")
            out = Q.topk_topp(xt, torch.tensor([v, v], device="cuda"), torch.tensor([0.3, 0.9], device="cuda", dtype=torch.float64),
                              flags=Q.TruncFlags(staged=staged), kept_count=kept, metrics=met)
            o = out.float().cpu().numpy()
            res = []
            for i in range(2):
                keep = oracle_keep_row(xs[i], v, [0.3, 0.9][i])
                res.append((int(keep.sum()), int(kept[i]), bool(np.array_equal(~np.isneginf(o[i]), keep))))
            m = Q.ops.decode_metrics(met)
            print(v, dt, "staged" if staged else Q.ops.pipeline_kind(xt), res, [(mm["trunc_hit"], mm["full_row_path"], mm["p_search_iters"]) for mm in m])
