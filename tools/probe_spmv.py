"""Profile driver: the fine-level SpMV and the l1-Jacobi smoother probes of
cfg2 inside cudaProfilerStart/Stop (for ncu --profile-from-start off)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2101_11649_b200 as mx  # noqa: E402

if os.environ.get("PROBE_CFG") == "cfg4":  # BASELINE cfg4 (frac_mgr_u_l1j)
    P = mx.frac_problem(64, seed=20210131)
    H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, mx.load_strategy("frac_mgr_u_l1j"),
                     P.unknown_map)
else:
    P = mx.mfd_problem(128, 128, 64, "layered", seed=20210129)
    H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, mx.load_strategy("mfd_mgr_pi_c1_l1j"))
names = sys.argv[1:] or ["spmv.A", "amg.0.resid", "amg.0.pre", "mgr.0.prolong"]
for nm in names:
    ms, by = H.time_kernel(nm, reps=20)
    print("avg20", nm, f"{ms * 1e3:.2f} us", f"{by / (ms * 1e-3) / 1e9:.0f} GB/s", flush=True)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for nm in names:
    ms, by = H.time_kernel(nm, reps=1)
    print(nm, ms, by / (ms * 1e-3) / 1e9, "GB/s")
torch.cuda.synchronize()
torch.cuda.profiler.stop()
