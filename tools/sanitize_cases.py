"""Small cases that exercise every synchronisation pattern of libmgrx, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
the low-sync GMRES (conditional graph + host loop), the MGS fused Arnoldi
kernel (grid barrier), its mailbox self-exchange, the single-CTA AMG tail,
the cluster dense solve (DSMEM flags) and the dense inverse, the sync-free,
block-partitioned and single-CTA Gauss-Seidel sweeps (NaN-sentinel polling),
BSR and SELL SpMV, and a 2-rank local-group shard (scattered setup)."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2101_11649_b200 as mx  # noqa: E402


def solve(P, name, ortho, rtol=1e-6):
    H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, mx.load_strategy(name), P.unknown_map)
    _, rep = H.solve(P.rhs, None, mx.KrylovConfig(restart=30, rel_tol=rtol, ortho=ortho))
    assert rep.converged, (name, ortho)
    return H


def main():
    which = sys.argv[1:] or ["all"]
    P = mx.mfd_problem(20, 20, 10, "iid")
    for o in ("cgs2", "mgs"):
        solve(P, "mfd_mgr_pi_c1_l1j", o)        # low-sync (graph) / fused MGS kernel, AMG tail
    solve(P, "mfd_mgr_pi_c1", "cgs2")           # single-CTA GS sweeps
    C = mx.comp_problem(10, 10, 6, wells=2)
    for o in ("cgs2", "mgs"):
        solve(C, "comp_mgr_l1j", o, 1e-5)       # dense inverse / cluster LU solve
    F = mx.frac_problem(8)
    solve(F, "frac_mgr_u_l1j", "cgs2")          # odd n
    if "all" in which or "large" in which:
        L = mx.mfd_problem(32, 32, 24, "layered")
        solve(L, "mfd_mgr_pi_c1", "cgs2")       # sync-free / block GS on the 24K-row level
    # 2-rank local group, scattered setup
    H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, mx.load_strategy("mfd_mgr_pi_c1_l1j"))
    st = mx.slab_row_starts(P, 2)
    g = mx.LocalGroup(2)
    with ThreadPoolExecutor(2) as ex:
        S = list(ex.map(lambda r: mx.Shard(H if r == 0 else None, r, 2, st, group=g, scatter=True, ctx=H.ctx),
                        range(2)))
        outs = list(ex.map(lambda s: s.solve(P.rhs[s.row_begin:s.row_end], None,
                                             mx.KrylovConfig(restart=30, rel_tol=1e-6)), S))
    assert all(o[1].converged for o in outs)
    for s in S:
        s.close()
    g.close()
    print("sanitize cases ok")


if __name__ == "__main__":
    main()
