"""CPU: the C-ABI library loads and exports exactly what include/qrita_b200.h declares; argument
validation happens before any CUDA call."""
import ctypes
import os
import re

import pytest

from paper_2602_01518_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "qrita_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(qrita_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(N.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    return N.load()


def test_header_declares_expected_entry_points():
    assert declared_functions() == sorted(N.EXPORTED_SYMBOLS)


def test_every_declared_symbol_is_exported(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_nm_exports_are_c_linkage():
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", N.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (qrita_\w+)", out))
    assert set(declared_functions()) <= exported


def test_metrics_struct_layout():
    assert ctypes.sizeof(N.RowMetricsC) == 40
    assert N.RowMetricsC.outlier_prob_sum.offset == 8


def test_workspace_bytes_and_strings(lib):
    assert lib.qrita_workspace_bytes(0, 10, 0, 0) == 0
    small = lib.qrita_workspace_bytes(1, 32000, 0, 0)
    big = lib.qrita_workspace_bytes(256, 128256, 0, 0)
    assert 0 < small < big
    # outlier scratch: 256 slots of 2 x uint32 per 1024-element chunk = 2 bytes per logit
    assert big < 256 * 128256 * 2.1
    assert lib.qrita_strerror(N.OK).decode() == "ok"
    assert "non-finite" in lib.qrita_strerror(N.ENONFINITE).decode()
    assert lib.qrita_version() >= 100


def test_argument_validation_without_gpu(lib):
    vp = ctypes.c_void_p
    # null pointers are rejected before any CUDA call
    rc = lib.qrita_topk_topp(vp(0), 8, 0, 1, 8, vp(0), vp(0), vp(0), 8, vp(0), vp(0), vp(0), 0, 0,
                             4096, vp(0))
    assert rc == N.EINVAL_ARG
    # bad dtype / flags / inplace mismatch with fake (never dereferenced) pointers
    fake = vp(0x1000)
    assert lib.qrita_topk_topp(fake, 8, 7, 1, 8, fake, fake, vp(0x2000), 8, vp(0), vp(0), fake, 1 << 20,
                               0, 4096, vp(0)) == N.EINVAL_ARG
    assert lib.qrita_topk_topp(fake, 8, 0, 1, 8, fake, fake, vp(0x2000), 8, vp(0), vp(0), fake, 1 << 20,
                               1 << 9, 4096, vp(0)) == N.EINVAL_ARG
    assert lib.qrita_topk_topp(fake, 8, 0, 1, 8, fake, fake, vp(0x2000), 8, vp(0), vp(0), fake, 1 << 20,
                               N.INPLACE, 4096, vp(0)) == N.EINVAL_ARG
    # ld < V
    assert lib.qrita_topk_topp(fake, 4, 0, 1, 8, fake, fake, vp(0x2000), 8, vp(0), vp(0), fake, 1 << 20,
                               0, 4096, vp(0)) == N.EINVAL_ARG
    # workspace too small
    assert lib.qrita_topk_topp(fake, 8, 0, 1, 8, fake, fake, vp(0x2000), 8, vp(0), vp(0), vp(0x100000),
                               16, 0, 4096, vp(0)) == N.EWORKSPACE


def test_product_has_no_oracle_dependency():
    pkg = os.path.join(ROOT, "paper_2602_01518_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import oracle|from oracle)", src, flags=re.M), f


def test_idx_and_host_entry_points_validate_before_cuda(lib):
    """qrita_topk_topp_idx / qrita_topk_topp_host / qrita_host_scratch_bytes: argument checks that
    return before any CUDA call (safe without a GPU)."""
    dummy = ctypes.c_void_p(256)
    V = 1000
    # neither masked output nor kept_idx
    assert lib.qrita_topk_topp_idx(dummy, V, 0, 4, V, dummy, dummy, None, V, None, V, dummy, None,
                                   dummy, 1 << 20, 0, 4096, None) == N.EINVAL_ARG
    # kept_idx narrower than V, or without kept_count / metrics to say how many entries are valid
    assert lib.qrita_topk_topp_idx(dummy, V, 0, 4, V, dummy, dummy, None, V, dummy, V - 1, dummy, None,
                                   dummy, 1 << 20, 0, 4096, None) == N.EINVAL_ARG
    assert lib.qrita_topk_topp_idx(dummy, V, 0, 4, V, dummy, dummy, None, V, dummy, V, None, None,
                                   dummy, 1 << 20, 0, 4096, None) == N.EINVAL_ARG
    # index-only output cannot be in place
    assert lib.qrita_topk_topp_idx(dummy, V, 0, 4, V, dummy, dummy, None, V, dummy, V, dummy, None,
                                   dummy, 1 << 20, N.INPLACE, 4096, None) == N.EINVAL_ARG
    # host pipeline: scratch size grows with B, covers both staging copies, rejects bad shapes
    s1 = lib.qrita_host_scratch_bytes(8, V, 0, 4)
    s2 = lib.qrita_host_scratch_bytes(16, V, 0, 4)
    assert s2 > s1 >= 2 * 8 * V * 4
    assert lib.qrita_host_scratch_bytes(8, V, 1, 4) < s1  # bf16 staging is half the size
    assert lib.qrita_host_scratch_bytes(0, V, 0, 4) == 0 and lib.qrita_host_scratch_bytes(8, V, 0, 0) == 0
    assert lib.qrita_topk_topp_host(dummy, 0, 8, V, dummy, dummy, dummy, None, None, dummy, s1, 0, 0, 4096,
                                    None) == N.EINVAL_ARG
    assert lib.qrita_topk_topp_host(dummy, 0, 8, V, dummy, dummy, dummy, None, None, dummy, s1 - 1, 4, 0, 4096,
                                    None) == N.EWORKSPACE
    assert lib.qrita_topk_topp_host(dummy, 0, 8, V, dummy, dummy, dummy, None, None, dummy, s1, 4, N.INPLACE,
                                    4096, None) == N.EINVAL_ARG
