"""Time the fused Arnoldi kernel at cfg2 size under MGRX_ARNOLDI_DBG flag
sets given on the command line (e.g. 0 32 2 34)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2101_11649_b200 as mx  # noqa: E402

P = mx.mfd_problem(128, 128, 64, "layered", seed=20210129)
H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, mx.load_strategy("mfd_mgr_pi_c1_l1j"))
H.solve(P.rhs, cfg=mx.KrylovConfig(restart=30, rel_tol=1e-6))
for dbg in sys.argv[1:]:
    os.environ["MGRX_ARNOLDI_DBG"] = dbg
    res = []
    for k in (9, 29):
        ms, by = H.time_kernel(f"arnoldi.{k}", reps=10)
        res.append(f"k={k}: {ms * 1e3:7.1f} us")
    print(os.environ.get("TAG", ""), "dbg", dbg, " | ".join(res), flush=True)
