"""Profiling driver: build BASELINE cfg2, set up the hierarchy, then run one
GMRES solve capped at --iters iterations inside cudaProfilerStart/Stop, so
`ncu --profile-from-start off` sees only solve-phase kernels."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2101_11649_b200 as mx  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--strategy", default="mfd_mgr_pi_c1")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--dims", default="128,128,64")
a = ap.parse_args()
nx, ny, nz = map(int, a.dims.split(","))
P = mx.mfd_problem(nx, ny, nz, "layered", seed=20210129)
H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, mx.load_strategy(a.strategy))
dev = torch.device("cuda", 0)
b = torch.from_numpy(P.rhs).to(dev)
x = torch.zeros(P.n, dtype=torch.float64, device=dev)
cfg = mx.KrylovConfig(restart=30, max_iters=a.iters, rel_tol=1e-6)
H.solve_device(b.data_ptr(), x.data_ptr(), cfg)  # warm-up: graph capture
x.zero_()
torch.cuda.synchronize()
torch.cuda.profiler.start()
rep = H.solve_device(b.data_ptr(), x.data_ptr(), cfg)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"iterations={rep.iterations} solve_s={rep.solve_s:.4f} launches={rep.gpu_launches}")
