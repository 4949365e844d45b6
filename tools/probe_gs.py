"""Time every AMG smoother sweep of the cfg2 hierarchy (probe kernels)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2101_11649_b200 as mx  # noqa: E402

strategy = sys.argv[1] if len(sys.argv) > 1 else "mfd_mgr_pi_c1"
P = mx.mfd_problem(128, 128, 64, "layered", seed=20210129)
H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, mx.load_strategy(strategy))
info = H.info()
tot = 0.0
out = []
for k in range(info["coarse_amg_levels"] - 1):
    for w in ("pre", "post"):
        ms, _ = H.time_kernel(f"amg.{k}.{w}", reps=10)
        tot += ms
        out.append(f"{k}.{w}={ms:.3f}")
print(os.environ.get("TAG", ""), "total_ms=%.3f" % tot, " ".join(out))
