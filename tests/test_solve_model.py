"""The whole-solve byte model (tools/solve_model.py) walks a
hierarchy through the dump grammar; checked here on the CPU oracle's
hierarchy (same grammar as the device one) against hand-summed terms."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import paper_2101_11649_b200 as mx  # noqa: E402
import refcpu  # noqa: E402
from solve_model import SolveModel, _spmv  # noqa: E402


def _ref(P, name):
    return refcpu.RefHierarchy(P.ptr, P.col, P.val, P.partition.field_order, P.partition.labels,
                               mx.load_strategy(name), P.unknown_map)


def test_mfd_model_terms():
    P = mx.mfd_problem(8, 8, 4, "iid")
    name = "mfd_mgr_pi_c1_l1j"
    R = _ref(P, name)
    sm = SolveModel(R, mx.load_strategy(name))
    # hand sum: one MGR level (jacobi F-relax, injection R) + 1 AMG V-cycle
    ptr, col, _, (n, _) = R.dump("mgr.0.A")
    F, C = R.dump("mgr.0.F"), R.dump("mgr.0.C")
    isf = np.zeros(n, bool)
    isf[F] = True
    rowf = np.repeat(isf, np.diff(ptr))
    nnz_cf = int(np.count_nonzero(~rowf & isf[col]))
    pptr = R.dump("mgr.0.P")[0]
    nf, nc = len(F), len(C)
    mgr = 24.0 * nf + 12.0 * nnz_cf + 4.0 * (nc + 1) + 8.0 * nf + 16.0 * nc
    mgr += 16.0 * nc + 12.0 * (int(pptr[-1]) - nc) + 4.0 * (nf + 1) + 8.0 * nc + 16.0 * nf
    info = R.info()
    amg = 0.0
    for k in range(info["coarse_amg_levels"]):
        a = R.dump(f"mgr.coarse.amg.{k}.A")
        m, nnz = a[3][0], int(a[0][-1])
        if k + 1 == info["coarse_amg_levels"]:
            amg += 8.0 * m * m + 24.0 * m
            break
        sweeps = 2 * (24.0 * m + _spmv(nnz, m, a[3][1]) + 16.0 * m)  # l1-Jacobi x2, pre + post
        p, r = R.dump(f"mgr.coarse.amg.{k}.P"), R.dump(f"mgr.coarse.amg.{k}.R")
        amg += sweeps + 2 * (_spmv(nnz, m, a[3][1]) + 8.0 * m)
        amg += _spmv(int(r[0][-1]), *r[3]) + _spmv(int(p[0][-1]), *p[3]) + 16.0 * m
    assert np.isclose(sm.m_prec, mgr + amg, rtol=0, atol=0.5)
    out = sm.solve_bytes(int(P.ptr[-1]), P.n, 35, 30)
    assert out["restart_cycles"] == 2
    assert out["bytes"] > 35 * (sm.m_prec + _spmv(int(P.ptr[-1]), P.n, P.n))
    # low-sync orthogonalisation: 16 n (k+3) per step instead of 24 n (k+1) + 32 n,
    # and no v0 scaling pass per cycle
    ls = sm.solve_bytes(int(P.ptr[-1]), P.n, 35, 30, ortho="cgs2")
    n = P.n
    mgs_orth = sum(24.0 * n * (k + 1) + 32.0 * n for k in list(range(30)) + list(range(5)))
    ls_orth = sum(16.0 * n * (k + 3) for k in list(range(30)) + list(range(5)))
    assert np.isclose(out["bytes"] - ls["bytes"], mgs_orth - ls_orth + 2 * 16.0 * n)


def test_comp_and_frac_models_run():
    for P, name in ((mx.comp_problem(6, 6, 4, wells=2), "comp_mgr_l1j"),
                    (mx.frac_problem(6), "frac_mgr_u_l1j")):
        R = _ref(P, name)
        sm = SolveModel(R, mx.load_strategy(name))
        assert sm.m_prec > 0
        assert sm.solve_bytes(int(P.ptr[-1]), P.n, 10, 30)["bytes"] > 0
