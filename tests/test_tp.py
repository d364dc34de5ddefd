"""Vocab-sharded (TP) variant, CPU side: shard bounds, workspace sizing and the C-ABI argument
checks of qrita_topk_topp_tp_comm (rejected before any CUDA call).  The protocol itself runs on the
GPU (tests/test_gpu_tp.py: threads-as-ranks on one GPU, gloo processes, NCCL)."""
import ctypes

import pytest

from paper_2602_01518_b200 import _native as N
from paper_2602_01518_b200.tp import QritaComm, shard_bounds


@pytest.fixture(scope="module")
def lib():
    return N.load()


def test_shard_bounds():
    assert shard_bounds(262144, 8) == [32768 * r for r in range(9)]
    b = shard_bounds(1000, 3)
    assert b[0] == 0 and b[-1] == 1000 and all(x < y for x, y in zip(b, b[1:]))


def test_tp_workspace_grows_with_world_and_kcap(lib):
    a = lib.qrita_tp_workspace_bytes(128, 32768, 0, 8, 1024)
    assert a > 0
    assert lib.qrita_tp_workspace_bytes(128, 32768, 0, 8, 64) < a
    assert lib.qrita_tp_workspace_bytes(128, 32768, 0, 2, 1024) < a
    assert lib.qrita_tp_workspace_bytes(0, 32768, 0, 8, 1024) == 0
    # k_cap above the shard width is clamped to it (at most V_r candidates per rank)
    assert lib.qrita_tp_workspace_bytes(4, 100, 0, 2, 10 ** 6) == lib.qrita_tp_workspace_bytes(4, 100, 0, 2, 100)


def test_tp_argument_checks(lib):
    comm = QritaComm()
    dummy = ctypes.c_void_p(256)

    def call(**kw):
        a = dict(B=4, Vr=100, Vg=200, off=0, kcap=10, flags=0, rank=0, world=2, comm=ctypes.addressof(comm),
                 out=dummy)
        a.update(kw)
        return lib.qrita_topk_topp_tp_comm(dummy, a["Vr"], 0, a["B"], a["Vr"], a["Vg"], a["off"], dummy, dummy,
                                           a["kcap"], a["out"], a["Vr"], None, dummy, 1 << 30, a["flags"],
                                           a["rank"], a["world"], ctypes.c_void_p(a["comm"]), None)

    assert call() == N.EINVAL_ARG              # the comm has no callbacks
    assert call(comm=0) == N.EINVAL_ARG
    assert call(rank=2) == N.EINVAL_ARG
    assert call(off=150) == N.EINVAL_ARG       # shard beyond V_global
    assert call(Vg=50) == N.EINVAL_ARG
    assert call(flags=N.SEARCH_BINARY) == N.EINVAL_ARG
    assert call(flags=N.INPLACE) == N.EINVAL_ARG  # inplace needs out == logits
    assert lib.qrita_topk_topp_tp(dummy, 100, 0, 4, 100, 200, 0, dummy, dummy, 10, dummy, 100, None, dummy,
                                  1 << 30, 0, 0, 2, None, None) == N.EINVAL_ARG
