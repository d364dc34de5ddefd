"""CPU: argument checks of the LM-head fusion API (no kernel runs) and its C-ABI arguments."""
import ctypes

import pytest
import torch

from paper_2602_01518_b200 import _native as N
from paper_2602_01518_b200.lmhead import lm_head_logits, lm_head_topk_topp


def test_host_tensors_rejected():
    h = torch.zeros(4, 64, dtype=torch.bfloat16)
    w = torch.zeros(100, 64, dtype=torch.bfloat16)
    with pytest.raises(TypeError):
        lm_head_logits(h, w)
    with pytest.raises(TypeError):
        lm_head_topk_topp(h, w, 5, 0.9)


def test_fp32_operands_rejected():
    with pytest.raises(TypeError):
        lm_head_logits(torch.zeros(4, 64), torch.zeros(100, 64))


def test_c_abi_argument_checks():
    lib = N.load()
    assert lib.qrita_lmhead_workspace_bytes(256, 128256) > lib.qrita_workspace_bytes(256, 128256, 0, 0)
    assert lib.qrita_lmhead_workspace_bytes(0, 10) == 0
    vp = ctypes.c_void_p
    # null operands, d not a multiple of 64, short leading dimensions: rejected before any CUDA call
    assert lib.qrita_lmhead_logits(vp(0), 64, vp(0), 64, 4, 100, 64, vp(0), 100, vp(0)) == N.EINVAL_ARG
    assert lib.qrita_lmhead_logits(vp(16), 64, vp(16), 64, 4, 100, 60, vp(16), 100, vp(0)) == N.EINVAL_ARG
    assert lib.qrita_lmhead_logits(vp(16), 32, vp(16), 64, 4, 100, 64, vp(16), 100, vp(0)) == N.EINVAL_ARG
    assert lib.qrita_lmhead_logits(vp(16), 64, vp(16), 64, 4, 100, 64, vp(16), 50, vp(0)) == N.EINVAL_ARG
    assert lib.qrita_lmhead_topk_topp(vp(16), 64, vp(16), 64, 4, 100, 64, vp(16), vp(16), vp(16), 100, vp(0), 100,
                                      vp(16), vp(0), vp(0), 0, 0, vp(0)) == N.EINVAL_ARG


def test_host_download_bytes_rule():
    """qrita_host_download_bytes (CPU, no CUDA call needed for plain host buffers): the sparse form for
    all-top-k batches with k <= 4096, dense rows otherwise."""
    import numpy as np
    lib = N.load()
    B, V = 8, 32000
    x = np.zeros((B, V), np.float32)
    o = np.zeros_like(x)
    k = np.full(B, 50, np.int64)
    k[3] = 1000
    vp = ctypes.c_void_p
    got = lib.qrita_host_download_bytes(B, V, 0, vp(k.ctypes.data), vp(x.ctypes.data), vp(o.ctypes.data))
    assert got == B * (1000 + 1) * 4
    k[5] = V                                  # a top-p-only row
    assert lib.qrita_host_download_bytes(B, V, 0, vp(k.ctypes.data), vp(x.ctypes.data),
                                         vp(o.ctypes.data)) == B * V * 4
    k[5] = 5000                               # above the sparse cap
    assert lib.qrita_host_download_bytes(B, V, 0, vp(k.ctypes.data), vp(x.ctypes.data),
                                         vp(o.ctypes.data)) == B * V * 4
