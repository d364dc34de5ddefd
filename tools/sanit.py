"""One small truncation case per invocation, for compute-sanitizer (tools/sanitize.sh):

    compute-sanitizer --tool racecheck python tools/sanit.py cfg2

Cases: cfg1; cfg2 (first 32 rows); cfg3 (4 rows, bf16, top-p only: distinct-value path); mixed (700
rows x 5000 with every mode, ties and an all-equal row: several rows per CTA); staged (V = 4999, the
unaligned 3-kernel pipeline); idx (kept-index output); nodup / binary / fallback ablations; tp
(the vocab-sharded protocol, 2 ranks as threads); host (the host-buffer pipeline, pageable); lmhead
(the LM-head GEMM with the fused streaming epilogue, in-kernel plans).
Each case checks its result against the oracle and prints "ok <case>"."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_01518_b200 as Q  # noqa: E402
from oracle.qrita_oracle import oracle_batch  # noqa: E402
from oracle.synth import bf16_bits_to_f32, config_inputs, to_bf16_bits  # noqa: E402


def mixed(b=700, v=5000, seed=4):
    r = np.random.default_rng(seed)
    x = r.normal(0, 1, (b, v)).astype(np.float32)
    x[::3] = np.round(x[::3] * 4) / 4
    x[7] = 0.25
    k = r.integers(1, 1025, b).astype(np.int64)
    p = r.uniform(0.3, 0.99, b)
    k[::5] = v
    p[1::5] = 1.0
    k[2::7] = v
    p[2::7] = 1.0
    return x, k, p


def check(x, got, k, p, label):
    want, _ = oracle_batch(x, k, p)
    got = np.asarray(got, dtype=np.float32)
    same = (got.view(np.uint32) == want.view(np.uint32)) | (np.isneginf(got) & np.isneginf(want))
    assert same.all(), f"{label}: rows {np.nonzero(~same.all(1))[0][:5]} differ"
    print("ok", label, flush=True)


def run(x, k, p, dtype=torch.float32, **flags):
    xt = torch.from_numpy(x).cuda().to(dtype)
    out = Q.topk_topp(xt, torch.from_numpy(k).cuda(), torch.from_numpy(p).cuda(),
                      flags=Q.TruncFlags(**flags) if flags else None, check=True)
    return out.float().cpu().numpy()


def main(case):
    if case in ("cfg1", "cfg2", "cfg3"):
        x, k, p, dt = config_inputs(case)
        n = {"cfg1": 1, "cfg2": 32, "cfg3": 4}[case]
        x, k, p = x[:n], k[:n], p[:n]
        check(x, run(x, k, p, torch.bfloat16 if dt == "bf16" else torch.float32), k, p, case)
    elif case == "mixed":
        x, k, p = mixed()
        check(x, run(x, k, p), k, p, case)
    elif case == "staged":
        x, k, p = mixed(96, 4999, 5)
        check(x, run(x, k, p, staged=True), k, p, case)
    elif case == "idx":
        x, k, p = mixed(64, 8192, 6)
        xt = torch.from_numpy(x).cuda()
        idx, cnt = Q.topk_topp_indices(xt, torch.from_numpy(k).cuda(), torch.from_numpy(p).cuda(), check=True)
        idx, cnt = idx.cpu().numpy(), cnt.cpu().numpy()
        got = np.full_like(x, -np.inf)
        for i in range(x.shape[0]):
            got[i, idx[i, :cnt[i]]] = x[i, idx[i, :cnt[i]]]
        check(x, got, k, p, case)
    elif case in ("binary", "fallback", "nosigma"):
        x, k, p = mixed(128, 4096, 7)
        fl = {"binary": dict(search="binary"), "fallback": dict(force_fallback=True),
              "nosigma": dict(use_sigma_trunc=False)}[case]
        check(x, run(x, k, p, **fl), k, p, case)
    elif case == "tp":
        from paper_2602_01518_b200.tp import simulate_tp
        x, k, p = mixed(32, 6000, 8)
        x = bf16_bits_to_f32(to_bf16_bits(x))
        for dt in (torch.float32, torch.bfloat16):
            out = simulate_tp(torch.from_numpy(x).cuda().to(dt), torch.from_numpy(k).cuda(),
                              torch.from_numpy(p).cuda(), world=2)
            check(x, out.float().cpu().numpy(), k, p, f"tp {dt}")
    elif case == "lmhead":
        from paper_2602_01518_b200.lmhead import lm_head_topk_topp
        g = torch.Generator().manual_seed(3)
        h = torch.randn(16, 128, generator=g).to(torch.bfloat16).cuda()
        w = (torch.randn(5000, 128, generator=g) / 128 ** 0.5).to(torch.bfloat16).cuda()
        _, k, p = mixed(16, 5000, 10)
        logits, idx, cnt = lm_head_topk_topp(h, w, torch.from_numpy(k), torch.from_numpy(p), check=True)
        x = logits.cpu().numpy()
        idx, cnt = idx.cpu().numpy(), cnt.cpu().numpy()
        got = np.full_like(x, -np.inf)
        for i in range(x.shape[0]):
            got[i, idx[i, :cnt[i]]] = x[i, idx[i, :cnt[i]]]
        check(x, got, k, p, case)
    elif case == "hostsparse":  # every row top-k: sparse downloads, host-built rows (pinned and pageable out)
        x, k, p = mixed(96, 8192, 11)
        k = np.minimum(k, 1000)
        for pin in (False, True):
            xh = torch.from_numpy(x)
            oh = torch.empty_like(xh)
            if pin:
                xh, oh = xh.pin_memory(), oh.pin_memory()
            out = Q.ops.topk_topp_host(xh, torch.from_numpy(k), torch.from_numpy(p), out=oh)
            check(x, out.numpy(), k, p, f"{case} pinned={pin}")
    elif case == "host":
        x, k, p = mixed(200, 8192, 9)
        out = Q.topk_topp(torch.from_numpy(x), torch.from_numpy(k), torch.from_numpy(p))
        check(x, out.numpy(), k, p, case)
    else:
        raise SystemExit(f"unknown case {case}")


if __name__ == "__main__":
    main(sys.argv[1])
