"""GPU: the native vocab-sharded protocol (qrita_topk_topp_tp) is bit-exact against the reference's
golden answers and the oracle.  Ranks share the one GPU: as threads of this process (simulate_tp,
ThreadComm), as gloo processes (TorchComm, host-staged exchange) and through NCCL at world 1."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import paper_2602_01518_b200 as Q
from oracle.qrita_oracle import oracle_batch
from oracle.synth import bf16_bits_to_f32, to_bf16_bits
from paper_2602_01518_b200.tp import shard_bounds, simulate_tp
from tests import golden_io as G

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _check(x, got, want, label):
    bad = np.nonzero(~G.same_bits(got, want).all(axis=1))[0]
    assert bad.size == 0, f"{label}: {bad.size} rows differ, first {bad[:5]}"


def test_cfg5_tp8_golden(cuda_device):
    x, k, p, _, trip, _ = G.config("cfg5")
    xt = torch.from_numpy(x).cuda()
    kc = torch.zeros(x.shape[0], dtype=torch.int32, device="cuda")
    out = simulate_tp(xt, torch.from_numpy(k).cuda(), torch.from_numpy(p).cuda(), world=8, kept_count=kc)
    _check(x, out.cpu().numpy(), G.masked_from_trip(x, trip), "cfg5 TP=8")
    assert np.array_equal(kc.cpu().numpy(), trip[:, 2])


def _mixed_case(seed, b, v, dtype):
    rng = np.random.default_rng(seed)
    x = rng.normal(0, 1, (b, v)).astype(np.float32)
    x[b // 2:] = np.round(x[b // 2:] * 4) / 4          # heavy ties in half of the rows
    x[1, :] = 0.5                                     # one all-equal row
    x[2, 5] = -0.0
    x[2, 9] = 0.0
    if dtype == torch.bfloat16:
        x = bf16_bits_to_f32(to_bf16_bits(x))
    k = rng.integers(1, 300, b).astype(np.int64)
    p = rng.uniform(0.3, 0.99, b)
    k[::4] = v                                        # top-p only
    p[1::4] = 1.0                                     # top-k only
    k[3], p[3] = v, 1.0                               # pass-through
    k[5] = v - 1
    p[6] = 1e-9
    return x, k, p


@pytest.mark.parametrize("world,dtype", [(2, torch.float32), (3, torch.float32), (4, torch.bfloat16),
                                         (8, torch.float32)])
def test_mixed_rows_vs_oracle(cuda_device, world, dtype):
    x, k, p = _mixed_case(11 + world, 24, 3000 + 7 * world, dtype)
    want, _ = oracle_batch(x, k, p)
    xt = torch.from_numpy(x).cuda().to(dtype)
    kc = torch.zeros(x.shape[0], dtype=torch.int32, device="cuda")
    out = simulate_tp(xt, torch.from_numpy(k).cuda(), torch.from_numpy(p).cuda(), world=world, kept_count=kc)
    _check(x, out.float().cpu().numpy(), want, f"mixed world={world} {dtype}")
    assert np.array_equal(kc.cpu().numpy(), (~np.isneginf(want)).sum(1))


@pytest.mark.parametrize("world", [16, 20])
def test_wide_candidate_rows(cuda_device, world):
    """world * k_cap candidates per row: 16 x 1000 takes the widest shared-memory sort (16384 slots),
    20 x 1000 the single-GPU kernels on column-ordered candidate rows."""
    rng = np.random.default_rng(77 + world)
    b, v = 6, 24000
    x = rng.normal(0, 1, (b, v)).astype(np.float32)
    x[3:] = np.round(x[3:] * 8) / 8                   # ties across shards
    k = np.array([1000, 999, 640, 1000, 17, 1000], dtype=np.int64)
    p = np.array([0.9, 1.0, 0.5, 0.999, 0.7, 1.0])
    want, _ = oracle_batch(x, k, p)
    out = simulate_tp(torch.from_numpy(x).cuda(), torch.from_numpy(k).cuda(), torch.from_numpy(p).cuda(),
                      world=world)
    _check(x, out.cpu().numpy(), want, f"wide world={world}")


def test_k_above_shard_width(cuda_device):
    """k larger than a shard (every rank sends its whole shard): the merge resolve's binary-search
    rank path instead of the merge tree (k exceeds the per-rank list slots)."""
    rng = np.random.default_rng(31)
    b, v = 10, 2000
    x = rng.normal(0, 1, (b, v)).astype(np.float32)
    x[6:] = np.round(x[6:] * 4) / 4                   # ties across shards
    k = np.array([1000, 400, 1999, 251, 600, 900, 1000, 333, 1500, 260], dtype=np.int64)
    p = np.array([0.9, 1.0, 0.95, 0.5, 0.99, 1.0, 0.8, 0.7, 1.0, 0.6])
    want, _ = oracle_batch(x, k, p)
    out = simulate_tp(torch.from_numpy(x).cuda(), torch.from_numpy(k).cuda(), torch.from_numpy(p).cuda(), world=8)
    _check(x, out.cpu().numpy(), want, "k above shard width")


def test_cfg3_rows_topp_only_bf16_tp4(cuda_device):
    x, k, p, _, trip, _ = G.config("cfg3")
    rows = slice(0, 8)
    xt = torch.from_numpy(x[rows]).cuda().to(torch.bfloat16)
    out = simulate_tp(xt, torch.from_numpy(k[rows]).cuda(), torch.from_numpy(p[rows]).cuda(), world=4)
    _check(x[rows], out.float().cpu().numpy(), G.masked_from_trip(x[rows], trip[rows]), "cfg3 rows TP=4")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_01518_b200.tp import TorchComm, topk_topp_tp
        x, k, p, _, trip, _ = G.config("cfg5")
        rows = slice(0, 32)
        x, k, p = x[rows], k[rows].copy(), p[rows].copy()
        k[::5] = x.shape[1]                           # some top-p-only rows too
        b = shard_bounds(x.shape[1], world)
        shard = torch.from_numpy(x[:, b[rank]:b[rank + 1]].copy()).cuda()
        comm = TorchComm()
        out = topk_topp_tp(shard, torch.from_numpy(k).cuda(), torch.from_numpy(p).cuda(), vocab_offset=b[rank],
                           vocab_size=x.shape[1], comm=comm, check=True)
        torch.cuda.synchronize()
        q.put((rank, out.cpu().numpy(), comm.bytes_exchanged))
    except BaseException as exc:
        q.put((rank, repr(exc), 0))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_processes_share_the_gpu(cuda_device, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = {}
    for _ in range(world):
        r, out, nbytes = q.get(timeout=600)
        assert not isinstance(out, str), out
        res[r] = (out, nbytes)
    for pr in procs:
        pr.join(timeout=120)
    x, k, p, _, trip, _ = G.config("cfg5")
    x, k, p = x[:32], k[:32].copy(), p[:32].copy()
    k[::5] = x.shape[1]
    want, _ = oracle_batch(x, k, p)
    got = np.concatenate([res[r][0] for r in range(world)], axis=1)
    _check(x, got, want, f"gloo world={world}")
    # partials only: far below the shard bytes (32 rows x 262144 / world x 4 B)
    assert res[0][1] < 32 * (262144 // world) * 4


def test_nccl_world1_subprocess(cuda_device):
    code = r'''
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, %r)
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=%r)
dist.init_process_group("gloo", rank=0, world_size=1)
import paper_2602_01518_b200 as Q
from paper_2602_01518_b200.tp import NcclComm, topk_topp_tp
x = torch.randn(16, 5000, device="cuda")
k = torch.randint(1, 200, (16,), device="cuda"); k[::3] = 5000
p = torch.rand(16, device="cuda", dtype=torch.float64) * 0.6 + 0.35
c = NcclComm()
a = topk_topp_tp(x, k, p, vocab_offset=0, vocab_size=5000, comm=c)
b = Q.topk_topp(x, k, p)
torch.cuda.synchronize()
same = (a.view(torch.int32) == b.view(torch.int32)).all().item()
c.close()
print("NCCL_OK" if same else "NCCL_MISMATCH")
''' % (ROOT, str(_free_port()))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert "NCCL_OK" in r.stdout, r.stdout + r.stderr
