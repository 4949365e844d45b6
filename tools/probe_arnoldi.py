"""Time the fused Arnoldi kernel at cfg2 size: full, rows-only, barrier-only;
with TRACE=1 also print one traced launch (per-phase globaltimer breakdown)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2101_11649_b200 as mx  # noqa: E402

P = mx.mfd_problem(128, 128, 64, "layered", seed=20210129)
H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, mx.load_strategy("mfd_mgr_pi_c1_l1j"))
H.solve(P.rhs, cfg=mx.KrylovConfig(restart=30, rel_tol=1e-6))
for dbg in ("0", "1", "2", "3"):
    os.environ["MGRX_ARNOLDI_DBG"] = dbg
    res = []
    for k in (0, 9, 29):
        ms, by = H.time_kernel(f"arnoldi.{k}", reps=10)
        res.append(f"k={k}: {ms * 1e3:7.1f} us ({by / ms / 1e6:6.0f} GB/s)")
    print(os.environ.get("TAG", ""), "dbg", dbg, " | ".join(res), flush=True)
if os.environ.get("TRACE"):
    os.environ["MGRX_ARNOLDI_DBG"] = os.environ.get("TRACE_DBG", "8")
    H.time_kernel("arnoldi.9", reps=1)
