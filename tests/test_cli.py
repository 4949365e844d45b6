"""CLI / bundle mirror (proj/tools/mgr_main.cpp, proj/src/bundle.cpp)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2101_11649_b200 as mx
from paper_2101_11649_b200 import cli

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bundle_roundtrip_text_and_binary(tmp_path):
    P = mx.comp_problem(6, 5, 4, wells=2)
    cli.write_bundle(P, str(tmp_path))
    for fn in ("matrix.mtx", "rhs.mtx", "labels.json", "meta.json", "bundle.npz"):
        assert (tmp_path / fn).exists()
    B = cli.read_bundle(str(tmp_path))  # binary sidecar (stamps match)
    assert np.array_equal(B.ptr, P.ptr) and np.array_equal(B.col, P.col) and np.array_equal(B.val, P.val)
    os.remove(tmp_path / "bundle.npz")
    T = cli.read_bundle(str(tmp_path))  # Matrix Market text, 17 significant digits round-trip
    assert np.array_equal(T.ptr, P.ptr) and np.array_equal(T.col, P.col)
    assert np.array_equal(T.val, P.val) and np.array_equal(T.rhs, P.rhs)
    assert T.partition.field_order == P.partition.field_order
    # a stale sidecar is ignored
    cli.write_bundle(P, str(tmp_path))
    with open(tmp_path / "rhs.mtx", "a") as f:
        f.write("\n")
    S = cli.read_bundle(str(tmp_path))
    assert np.array_equal(S.rhs, P.rhs)


def test_mm_reader_sums_duplicates_in_order(tmp_path):
    p = tmp_path / "m.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n1 1 2.0\n2 2 5.0\n")
    ptr, col, val, shape = cli.mm_read(str(p))
    assert list(ptr) == [0, 1, 2] and list(val) == [3.0, 5.0]


def test_usage_errors_exit_2(tmp_path):
    assert cli.main(["solve", "--bundle", str(tmp_path / "nope"), "--strategy", "mfd_mgr_pi"]) == 2
    P = mx.mfd_problem(3, 3, 2, "iid")
    cli.write_bundle(P, str(tmp_path / "b"))
    assert cli.main(["solve", "--bundle", str(tmp_path / "b"), "--strategy", "no_such_strategy"]) == 2
    assert cli.main(["solve", "--bundle", str(tmp_path / "b"), "--strategy", "comp_mgr"]) == 2  # unknown field
    assert cli.main(["study", "--problem", "mfd", "--sizes", "4,x", "--strategies", "mfd_mgr_pi"]) == 2


@pytest.mark.gpu
def test_cli_solve_on_gpu(tmp_path):
    assert cli.main(["generate", "--problem", "mfd", "--config", "cfg1", "--out", str(tmp_path / "b")]) == 0
    rc = cli.main(["solve", "--bundle", str(tmp_path / "b"), "--strategy", "mfd_mgr_pi", "--tol", "1e-6",
                   "--restart", "30", "--out", str(tmp_path / "o")])
    assert rc == 0
    head, row = (tmp_path / "o" / "report.csv").read_text().strip().split("\n")
    assert head == cli.CSV_HEADER
    rep = json.loads((tmp_path / "o" / "report.json").read_text())
    assert rep["converged"] and rep["true_residual"] <= 1e-6 and rep["dofs"] == 16800
    x = cli.mm_read_vector(str(tmp_path / "o" / "x.mtx"))
    assert x.size == 16800


@pytest.mark.gpu
@pytest.mark.parametrize("problem,sizes,strategies,tol,ceiling", [
    ("mfd", "8,16,32", "mfd_mgr_pi,mfd_mgr_pi_c1_l1j", 1e-7, 30),   # SPEC.md:750 criterion 6 (TPFA, MGR_pi)
    ("comp", "8,12,16", "comp_mgr,comp_mgr_l1j", 1e-6, 40),           # criterion 7 (2 wells)
    ("frac", "8,12,16", "frac_mgr_u,frac_mgr_u_l1j", 1e-6, 60),      # criterion 8 (MGR_U, ratio <= 1.5)
])
def test_cli_study_mesh_independence_on_gpu(tmp_path, problem, sizes, strategies, tol, ceiling):
    """The `study` mirror (proj/tools/mgr_main.cpp:344-400) on the GPU path: every
    refinement converges, iteration counts stay under the SPEC ceilings and the
    max/min growth ratio per strategy is <= 1.5."""
    rc = cli.main(["study", "--problem", problem, "--sizes", sizes, "--strategies", strategies, "--tol", str(tol),
                   "--restart", "30", "--out", str(tmp_path)])
    assert rc == 0
    out = json.loads((tmp_path / "study.json").read_text())
    assert len(out["rows"]) == len(sizes.split(",")) * len(strategies.split(","))
    for r in out["rows"]:
        assert r["converged"] and r["iterations"] <= ceiling, r
    for s, g in out["growth"].items():
        assert g is not None and g <= 1.5, (s, g, [r["iterations"] for r in out["rows"] if r["strategy"] == s])
    assert (tmp_path / "study.csv").read_text().count("growth,") == len(strategies.split(","))
