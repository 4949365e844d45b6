"""CPU tests of the refcpu oracle: the ported known-answer pins, the golden
fixtures it produced at commit time, and its behaviour on the BASELINE cfg1
system (iteration ceilings of SPEC.md:750-760)."""
import json
import os
import subprocess

import numpy as np
import pytest

import refcpu
import paper_2101_11649_b200 as mx

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_pins_binary_passes():
    refcpu.build()
    out = subprocess.run([refcpu.PINS], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 failures" in out.stdout


def test_oracle_spmv_matches_row_order():
    rng = np.random.default_rng(0)
    n = 50
    ptr = [0]
    col, val = [], []
    for i in range(n):
        cs = sorted(rng.choice(n, size=rng.integers(1, 8), replace=False))
        col += cs
        val += list(rng.standard_normal(len(cs)))
        ptr.append(len(col))
    x = rng.standard_normal(n)
    y = refcpu.spmv(ptr, col, val, x)
    for i in range(n):
        s = 0.0
        for k in range(ptr[i], ptr[i + 1]):
            s += val[k] * x[col[k]]
        assert y[i] == s


@pytest.mark.parametrize("strategy,ceiling", [("mfd_mgr_pi", 30), ("mfd_mgr_pi_c1", 30),
                                              ("mfd_mgr_pi_c1_l1j", 30), ("mfd_mgr_p", 40)])
def test_oracle_cfg1_converges(strategy, ceiling):
    P = mx.mfd_problem(20, 20, 10, "iid", seed=20210128)
    H = refcpu.RefHierarchy(P.ptr, P.col, P.val, P.partition.field_order, P.partition.labels,
                            mx.load_strategy(strategy))
    x, rep = H.solve(P.rhs, restart=30, rel_tol=1e-6)
    assert rep["converged"] and rep["iterations"] <= ceiling
    import scipy.sparse as sp
    A = sp.csr_matrix((P.val, P.col, P.ptr), shape=(P.n, P.n))
    assert np.linalg.norm(P.rhs - A @ x) <= 1e-6 * np.linalg.norm(P.rhs)


def _golden_cases():
    with open(os.path.join(GOLDEN, "oracle_golden.json")) as f:
        return json.load(f)["cases"]


@pytest.mark.parametrize("case", _golden_cases(), ids=lambda c: c["id"])
def test_oracle_matches_golden(case):
    """The oracle reproduces the fixtures committed by tests/golden/make_golden.py
    (hierarchy digests and residual history)."""
    import make_golden

    got = make_golden.run_case(case["spec"])
    assert got["shape"] == case["shape"]
    assert got["digests"] == case["digests"]
    assert got["iterations"] == case["iterations"]
    h0, h1 = np.array(got["history"]), np.array(case["history"])
    assert h0.shape == h1.shape and np.allclose(h0, h1, rtol=1e-12, atol=0)


def test_oracle_errors_name_rows():
    # zero diagonal in the F block -> diag_inverse names the A_FF row
    ptr = np.array([0, 2, 4, 5], np.int32)
    col = np.array([0, 1, 0, 1, 2], np.int32)
    val = np.array([1.0, 1.0, 1.0, 0.0, 2.0])
    with pytest.raises(refcpu.RefError, match="zero diagonal entry at row 1"):
        refcpu.RefHierarchy(ptr, col, val, ["a", "b"], [0, 0, 1],
                            json.dumps({"levels": [{"f_fields": ["a"]}], "coarse": {"kind": "dense_lu"}}))
    with pytest.raises(refcpu.RefError, match="unknown key 'bogus'"):
        refcpu.RefHierarchy(ptr, col, val, ["a", "b"], [0, 0, 1], '{"bogus": 1}')
    with pytest.raises(refcpu.RefError) as e:
        refcpu.RefHierarchy(ptr, col, val, ["a", "b"], [0, 0, 1],
                            json.dumps({"levels": [{"f_fields": ["a"]}, {"f_fields": ["a"]}]}))
    assert e.value.code == 2 and "eliminated twice" in str(e.value)


def test_oracle_solve_op_with_own_operator_is_solve():
    """ref_solve_op (gmres with the operator passed apart from the hierarchy,
    proj/include/mgrkit/krylov.hpp:33-34) on the hierarchy's own A is ref_solve,
    bit for bit; on a perturbed operator it still converges to that operator's
    solution."""
    P = mx.mfd_problem(6, 5, 4, "iid")
    text = mx.load_strategy("mfd_mgr_pi_c1")
    R = refcpu.RefHierarchy(P.ptr, P.col, P.val, P.partition.field_order, P.partition.labels, text)
    x, rep = R.solve(P.rhs, restart=30, rel_tol=1e-8)
    xo, repo = R.solve_op(P.ptr, P.col, P.val, P.rhs, restart=30, rel_tol=1e-8)
    assert rep["history"] == repo["history"] and np.array_equal(x, xo)
    val1 = P.val * (1.0 + 0.02 * np.random.default_rng(3).uniform(-1.0, 1.0, P.val.size))
    x1, rep1 = R.solve_op(P.ptr, P.col, val1, P.rhs, restart=30, rel_tol=1e-8)
    assert rep1["converged"] and rep1["iterations"] >= rep["iterations"]
    y = refcpu.spmv(P.ptr, P.col, val1, x1)
    assert np.linalg.norm(P.rhs - y) <= 1e-8 * np.linalg.norm(P.rhs) * (1 + 1e-9)
