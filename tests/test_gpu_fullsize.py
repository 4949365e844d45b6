"""Parity at the BASELINE configs' full sizes, against the refcpu oracle.

Cases: cfg2 4.2M DOF, cfg3 2.0M DOF, cfg4 0.78M DOF /
60M nnz, cfg5's 1-GPU point 4.2M DOF, each with its l1-Jacobi strategy (the
bench's) AND the reference's shipped Gauss-Seidel strategy verbatim
(`mfd_mgr_pi` with 8 V-cycles, `comp_mgr`, `frac_mgr_u`; proj/strategies/).

Per case (north_star bar, BASELINE.json):
* setup: every hierarchy operator (A, P, R at every level) and every C/F
  splitting of the device setup bit-exact against the oracle;
* the device solve in the reference's orthogonalisation (``ortho="mgs"``)
  and the oracle in the canonical reduction order agree bit for bit on the
  first 10 residual-history entries;
* against the oracle run TO CONVERGENCE in an independent inner-product order
  (``sequential``: one accumulator, left to right; the device never uses
  it): history within 1e-10 relative for the first 10 entries, iterations
  within +-1, and the device's final true residual (recomputed on the host)
  within rtol; the same 1e-10 bar against Eigen's SSE2 packet order on the
  first 10 entries;
* the same bar for the default low-synchronisation orthogonalisation
  (``ortho="cgs2"``) against the converged sequential-order oracle.
"""
import os

import numpy as np
import pytest
import scipy.sparse as sp

import paper_2101_11649_b200 as mx
import refcpu

pytestmark = pytest.mark.gpu

MFD2 = lambda: mx.mfd_problem(128, 128, 64, "layered", sigma=1.5, seed=20210129)  # noqa: E731
COMP3 = lambda: mx.comp_problem(100, 100, 50, wells=8, seed=20210130)  # noqa: E731
FRAC4 = lambda: mx.frac_problem(64, seed=20210131)  # noqa: E731
COMP5 = lambda: mx.comp_problem(128, 128, 64, wells=16, seed=20210134)  # noqa: E731

CASES = {
    "cfg2_l1j": (MFD2, "mfd_mgr_pi_c1_l1j", 1e-6),
    "cfg2_gs8": (MFD2, "mfd_mgr_pi", 1e-6),  # shipped strategy verbatim: 8 V-cycles, hybrid GS
    "cfg3_l1j": (COMP3, "comp_mgr_l1j", 1e-5),
    "cfg3_gs": (COMP3, "comp_mgr", 1e-5),
    "cfg4_l1j": (FRAC4, "frac_mgr_u_l1j", 1e-6),
    "cfg4_gs": (FRAC4, "frac_mgr_u", 1e-6),
    "cfg5_l1j": (COMP5, "comp_mgr_l1j", 1e-5),
}
K = 10  # history entries under the north_star bar


def _same(a, b):
    if isinstance(a, tuple):
        return (a[3] == b[3] and np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
                and np.array_equal(a[2].view(np.int64), b[2].view(np.int64)))
    if a.dtype == np.float64:
        return np.array_equal(a.view(np.int64), b.view(np.int64))
    return np.array_equal(a, b)


def within_bar(h, hr, k=K):
    """1e-10 relative to the residual scale max(|r_k|, |r_0|), r_0 / ||b|| = 1
    (zero initial guess), on the first k entries (tests/test_gpu_parity.py:
    history_close explains the scale)."""
    k = min(k, len(h), len(hr))
    h, hr = np.asarray(h[:k]), np.asarray(hr[:k])
    return bool(np.all(np.abs(h - hr) <= 1e-10 * np.maximum(np.abs(hr), 1.0)))


@pytest.mark.parametrize("case", list(CASES))
def test_fullsize_parity(case):
    make, strategy, rtol = CASES[case]
    P = make()
    text = mx.load_strategy(strategy)
    refcpu.set_threads(os.cpu_count() or 1)
    R = refcpu.RefHierarchy(P.ptr, P.col, P.val, P.partition.field_order, P.partition.labels, text, P.unknown_map)
    H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, text, P.unknown_map)
    assert H.info() == R.info()
    for path in refcpu.dump_paths(R.info()):
        assert _same(H.dump(path), R.dump(path)), f"{case}: {path} differs from the oracle"
    M = sp.csr_matrix((P.val, P.col, P.ptr), shape=(P.n, P.n))
    bnorm = np.linalg.norm(P.rhs)

    # device solves: the reference's MGS (bitwise mode) and the default
    x_m, rep_m = H.solve(P.rhs, None, mx.KrylovConfig(restart=30, rel_tol=rtol, ortho="mgs"))
    x_c, rep_c = H.solve(P.rhs, None, mx.KrylovConfig(restart=30, rel_tol=rtol, ortho="cgs2"))
    for x, rep in ((x_m, rep_m), (x_c, rep_c)):
        assert rep.converged, (case, rep)
        assert np.linalg.norm(P.rhs - M @ x) <= rtol * bnorm * (1 + 1e-9), case

    try:
        # canonical order: bitwise on the first K entries (MGS mode)
        refcpu.set_dot_order("canonical")
        _, r_can = R.solve(P.rhs, restart=30, max_iters=K, rel_tol=rtol)
        k = min(K, len(r_can["history"]))
        assert rep_m.residual_history[:k] == r_can["history"][:k], case
        # Eigen's SSE2 order: the 1e-10 bar on the first K entries
        refcpu.set_dot_order("eigen_sse2")
        _, r_eig = R.solve(P.rhs, restart=30, max_iters=K, rel_tol=rtol)
        assert within_bar(rep_m.residual_history, r_eig["history"]), case
        assert within_bar(rep_c.residual_history, r_eig["history"]), case
        # sequential order, run to convergence: 1e-10 bar, iterations +-1
        refcpu.set_dot_order("sequential")
        x_s, r_seq = R.solve(P.rhs, restart=30, rel_tol=rtol)
    finally:
        refcpu.set_dot_order("canonical")
    assert r_seq["converged"], case
    assert np.linalg.norm(P.rhs - M @ x_s) <= rtol * bnorm * (1 + 1e-9), case
    for rep in (rep_m, rep_c):
        assert within_bar(rep.residual_history, r_seq["history"]), (case, rep.residual_history[:K],
                                                                     r_seq["history"][:K])
        assert abs(rep.iterations - r_seq["iterations"]) <= 1, (case, rep.iterations, r_seq["iterations"])
