"""Cold-L2 ("cold:" differential) and warm probe times of cfg2 hierarchy
operators, for A/B runs under MGRX_* environment knobs.
    python tools/probe_cold.py amg.1.resid amg.1.pre ..."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2101_11649_b200 as mx  # noqa: E402

P = mx.mfd_problem(128, 128, 64, "layered", seed=20210129)
H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, mx.load_strategy("mfd_mgr_pi_c1_l1j"))
x, rep = H.solve(P.rhs, None, mx.KrylovConfig(restart=30, rel_tol=1e-6))
for _ in range(3):
    x, rep = H.solve(P.rhs, None, mx.KrylovConfig(restart=30, rel_tol=1e-6))
print("solve_ms", f"{rep.solve_s * 1e3:.2f}", "its", rep.iterations, flush=True)
names = sys.argv[1:] or ["amg.1.resid", "amg.1.pre", "amg.1.post", "amg.0.resid", "amg.0.pre", "amg.2.resid",
                         "amg.2.pre", "mgr.0.rres", "precond.inexact"]
for nm in names:
    ms, by = H.time_kernel(nm, reps=20)
    msc, _ = H.time_kernel("cold:" + nm, reps=20)
    print("probe", nm, f"warm {ms * 1e3:.2f} us", f"cold {msc * 1e3:.2f} us", flush=True)
