"""Row-sharded multi-GPU plumbing (BASELINE cfg4): contiguous row blocks, the
per-rank split bench.py uses, the max-over-ranks job time, and the gathered result — on CPU with
world-size-2 gloo and the oracle standing in for the CUDA op (the split is under test here; the
kernels' sharded runs are in tests/test_gpu_sharded.py)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.qrita_oracle import oracle_batch
from paper_2602_01518_b200.sharded import aggregate_max, gather_rows, rank_rows, row_blocks

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("b,n", [(1024, 1), (1024, 2), (1024, 8), (7, 3), (3, 8), (256, 5)])
def test_row_blocks_cover_contiguously(b, n):
    blocks = row_blocks(b, n)
    assert len(blocks) == n and blocks[0][0] == 0 and blocks[-1][1] == b
    for (lo0, hi0), (lo1, _) in zip(blocks, blocks[1:]):
        assert hi0 == lo1
    sizes = [hi - lo for lo, hi in blocks]
    assert max(sizes) - min(sizes) <= 1
    assert rank_rows(b, n - 1, n) == blocks[-1]
    with pytest.raises(ValueError):
        rank_rows(b, n, n)


def test_bench_rank_block_generation_matches_full_matrix():
    sys.path.insert(0, ROOT)
    from bench import _normal_rows
    full = np.random.default_rng(4).normal(0.0, 1.0, (10, 300)).astype(np.float32)
    parts = [_normal_rows(4, 10, 300, lo, hi, chunk=3) for lo, hi in row_blocks(10, 4)]
    assert np.array_equal(np.concatenate(parts), full)


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
    lo, hi = rank_rows(x.shape[0], rank, world)
    out, _ = oracle_batch(x[lo:hi], k[lo:hi], p[lo:hi])      # stand-in for the CUDA op
    full = gather_rows(torch.from_numpy(out), x.shape[0])
    job = aggregate_max(float(10 + rank))                     # per-rank "time"
    q.put((rank, (lo, hi), full.numpy(), job))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_row_sharded_split_and_aggregate(world):
    rng = np.random.default_rng(7)
    b, v = 11, 500
    x = rng.normal(0, 1, (b, v)).astype(np.float32)
    k = rng.integers(1, 60, b).astype(np.int64)
    p = rng.uniform(0.5, 0.99, b)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, x, k, p, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict((r, rest) for r, *rest in (q.get(timeout=300) for _ in range(world)))
    for pr in procs:
        pr.join(timeout=60)
    want, _ = oracle_batch(x, k, p)
    spans = sorted(res[r][0] for r in range(world))
    assert spans[0][0] == 0 and spans[-1][1] == b
    for r in range(world):
        full, job = res[r][1], res[r][2]
        same = (full.view(np.uint32) == want.view(np.uint32)) | (np.isneginf(full) & np.isneginf(want))
        assert same.all()
        assert job == 10 + world - 1        # max over ranks


def test_bench_gpus_without_gpus_fails_loudly():
    if torch.cuda.device_count() >= 2:
        pytest.skip("this host has 2 GPUs")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 2
    assert "needs 2 visible GPUs" in r.stderr
