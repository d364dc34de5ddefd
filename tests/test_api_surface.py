"""CPU: the drop-in surface — every public name of the reference package exists with the
reference's defaults, the QRTL / CSV formats are byte-compatible, the report schema matches, and
the CLI's flag / I/O error paths return the reference's exit codes (no GPU needed for any of it)."""
import inspect
import os
import sys

import numpy as np
import pytest

import paper_2602_01518_b200 as Q
from paper_2602_01518_b200 import cli

REF_SRC = "/root/reference/pkg/src"


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference tree not mounted (GPU box)")
    sys.path.insert(0, REF_SRC)
    import sigmatop
    return sigmatop


def test_every_reference_name_is_exported(ref):
    missing = [n for n in ref.__all__ if not hasattr(Q, n)]
    assert missing == []


def test_signatures_keep_reference_parameters(ref):
    for name in ("run_batch", "verify_batch", "bench", "synth_batch", "truncate_topk", "truncate_topp",
                 "truncate_topk_topp", "row_stats", "gather_outliers", "lookup_delta_topk", "lookup_delta_topp",
                 "threshold_from", "is_hit", "quaternary_topk", "quaternary_topp", "binary_topk", "binary_topp",
                 "oracle_topk", "oracle_topp", "oracle_topk_topp", "read_logits", "write_logits",
                 "read_targets_csv", "write_targets_csv", "write_report_csv", "generate_table"):
        rp = list(inspect.signature(getattr(ref, name)).parameters)
        op = list(inspect.signature(getattr(Q, name)).parameters)
        assert op[:len(rp)] == rp, (name, rp, op)


def test_tables_are_the_reference_tables(ref):
    assert np.array_equal(Q.TOPK_TABLE.entries, ref.TOPK_TABLE.entries)
    assert np.array_equal(Q.TOPP_TABLE.entries, ref.TOPP_TABLE.entries)


def test_scalar_sigma_arithmetic_matches(ref):
    st = Q.GaussianStats(0.013, 1.07, 4096)
    rst = ref.GaussianStats(0.013, 1.07, 4096)
    for v in (7, 1000, 128256):
        for k in sorted({1, 2, v // 3, v - 1, v}):
            assert Q.lookup_delta_topk(k, v) == ref.lookup_delta_topk(k, v)
            d = Q.lookup_delta_topk(k, v)
            assert Q.threshold_from(st, d) == Q.TruncThreshold(**vars(ref.threshold_from(rst, d)))
    for p in (1e-9, 0.1, 0.5, 0.9, 0.95, 0.999, 1.0):
        assert Q.lookup_delta_topp(p) == ref.lookup_delta_topp(p)
    with pytest.raises(ValueError):
        Q.lookup_delta_topk(0, 10)
    with pytest.raises(ValueError):
        Q.lookup_delta_topp(1.5)


def test_qrtl_and_targets_roundtrip_with_reference(ref, tmp_path):
    x = np.random.default_rng(1).normal(size=(3, 17)).astype(np.float32)
    x[1, 2] = -np.inf
    a, b = tmp_path / "a.qrtl", tmp_path / "b.qrtl"
    Q.write_logits(x, a)
    ref.write_logits(ref.LogitBatch(np.where(np.isinf(x), 0, x).astype(np.float32)), b)
    assert a.read_bytes()[:16] == b.read_bytes()[:16]
    back = ref.read_logits(a).values
    assert np.array_equal(back.view(np.uint32), x.view(np.uint32))
    assert np.array_equal(Q.read_logits(b).values, ref.read_logits(b).values)
    t = Q.TruncTargets(np.array([1, 5, 17]), np.array([0.1, 0.9, 1.0]))
    Q.write_targets_csv(t, tmp_path / "t.csv")
    rt = ref.read_targets_csv(tmp_path / "t.csv")
    assert np.array_equal(rt.k, t.k) and np.array_equal(rt.p, t.p)
    ref.write_targets_csv(rt, tmp_path / "r.csv")
    assert (tmp_path / "r.csv").read_bytes() == (tmp_path / "t.csv").read_bytes()


def test_qrtl_errors(tmp_path):
    p = tmp_path / "bad.qrtl"
    p.write_bytes(b"QRTX" + bytes(12))
    with pytest.raises(ValueError, match="bad magic"):
        Q.read_logits(p)
    p.write_bytes(b"QR")
    with pytest.raises(ValueError, match="truncated header"):
        Q.read_logits(p)
    import struct
    p.write_bytes(struct.pack("<4sIII", b"QRTL", 1, 2, 3) + bytes(8))
    with pytest.raises(ValueError, match="payload bytes"):
        Q.read_logits(p)
    (tmp_path / "t.csv").write_text("row,k,p\n1,5,0.5\n")
    with pytest.raises(ValueError, match="consecutive"):
        Q.read_targets_csv(tmp_path / "t.csv")


def test_report_schema(ref, tmp_path):
    assert Q.REPORT_COLUMNS == ref.engine.REPORT_COLUMNS
    rows = [{"run_id": "A", "B": 2, "V": 8, "wall_ms": 1.5}]
    Q.write_report_csv(rows, tmp_path / "a.csv")
    ref.write_report_csv(rows, tmp_path / "b.csv")
    assert (tmp_path / "a.csv").read_bytes() == (tmp_path / "b.csv").read_bytes()


def test_cli_exit_codes_without_gpu(tmp_path):
    assert cli.main(["bench", "--repeats", "2"]) == cli.EXIT_BAD_FLAGS
    assert cli.main(["verify", "--exhaustive", "--vocab", "9"]) == cli.EXIT_BAD_FLAGS
    assert cli.main(["run", "--input", str(tmp_path / "missing.qrtl")]) == cli.EXIT_IO
    with pytest.raises(SystemExit):
        cli.main(["run", "--k", "0"])
