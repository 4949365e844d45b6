"""Per-level Gauss-Seidel sweep times of the cfg2 GS variant (mfd_mgr_pi_c1):
amg.<k>.pre / .post probes (exact sequential forward / backward sweeps)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2101_11649_b200 as mx  # noqa: E402

P = mx.mfd_problem(128, 128, 64, "layered", seed=20210129)
H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, mx.load_strategy("mfd_mgr_pi_c1"))
info = H.info()
for k in range(info["coarse_amg_levels"] - 1):
    for w in ("pre", "post", "resid"):
        ms, by = H.time_kernel(f"amg.{k}.{w}", reps=5)
        print(f"amg.{k}.{w} {ms * 1e3:9.1f} us", flush=True)
