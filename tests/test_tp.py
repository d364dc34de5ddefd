"""Vocab-sharded (TP) protocol: world-size-2 gloo on CPU with the oracle as the local op (the
protocol, not the kernels, is under test here), plus the single-GPU simulation at cfg5 size."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.qrita_oracle import oracle_batch


def cpu_op(x, k, p):
    out, _ = oracle_batch(x.numpy(), k.numpy(), p.numpy())
    return torch.from_numpy(out)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, x, k, p, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2602_01518_b200.tp import topk_topp_tp
    v = x.shape[1]
    bounds = [v * r // world for r in range(world + 1)]
    shard = torch.from_numpy(x[:, bounds[rank]:bounds[rank + 1]].copy())
    out = topk_topp_tp(shard, torch.from_numpy(k), torch.from_numpy(p), vocab_offset=bounds[rank],
                       vocab_size=v, op=cpu_op)
    q.put((rank, out.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def _run(world, x, k, p):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, x, k, p, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
    return np.concatenate([res[r] for r in range(world)], axis=1)


def _same(a, b):
    return ((a.view(np.uint32) == b.view(np.uint32)) | (np.isneginf(a) & np.isneginf(b))).all()


def test_tp_gloo_world2_matches_unsharded():
    rng = np.random.default_rng(5)
    b, v = 12, 1001
    x = rng.normal(size=(b, v)).astype(np.float32)
    x[3] = np.round(x[3] * 2)                     # heavy ties across the shard boundary
    x[4, :] = 1.0                                 # all equal
    k = rng.integers(1, 300, size=b).astype(np.int64)
    k[5] = v                                      # top-p only row (gathered path)
    k[6] = v - 1
    p = rng.uniform(0.3, 0.99, size=b)
    p[7] = 1.0                                    # top-k only
    got = _run(2, x, k, p)
    want, _ = oracle_batch(x, k, p)
    assert _same(got, want)


def test_tp_simulated_world8_cpu():
    from paper_2602_01518_b200.tp import simulate_tp
    rng = np.random.default_rng(6)
    x = rng.normal(size=(6, 3000)).astype(np.float32)
    k = np.array([1, 10, 500, 2999, 3000, 77], dtype=np.int64)
    p = np.array([0.9, 1.0, 0.5, 0.95, 0.7, 0.999])
    got = simulate_tp(torch.from_numpy(x), torch.from_numpy(k), torch.from_numpy(p), 8, op=cpu_op).numpy()
    want, _ = oracle_batch(x, k, p)
    assert _same(got, want)


@pytest.mark.gpu
def test_tp_simulated_cfg5_on_gpu(cuda_device):
    from paper_2602_01518_b200.tp import simulate_tp
    from tests import golden_io as G
    x, k, p, _, trip, _ = G.config("cfg5")
    out = simulate_tp(torch.from_numpy(x).cuda(), torch.from_numpy(k).cuda(), torch.from_numpy(p).cuda(), 8)
    got = out.cpu().numpy()
    want = G.masked_from_trip(x, trip)
    assert G.same_bits(got, want).all()
