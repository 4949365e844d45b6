"""Run one roofline probe of bench.py's hierarchy under a profiler window
(cudaProfilerStart/Stop), for `ncu --set full --profile-from-start off`:

    ncu --set full --clock-control none --import-source on --profile-from-start off \
        -o gpurun_out/x python tools/ncu_probe.py cfg2 spmv.A

Only the probe's launches (time_kernel with reps=1) are inside the window."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2101_11649_b200 as mx  # noqa: E402


def main():
    cfg, names = sys.argv[1], sys.argv[2:]
    bench.CONFIG = cfg
    bench.STRATEGY = bench.CONFIGS[cfg]["strategy"]
    bench.RTOL = bench.CONFIGS[cfg]["rtol"]
    P = bench.make_problem()
    H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, mx.load_strategy(bench.STRATEGY), P.unknown_map)
    H.solve(P.rhs, None, mx.KrylovConfig(restart=30, rel_tol=bench.RTOL))  # warm (work vectors, plans)
    for nm in names:
        H.time_kernel(nm, reps=2)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for nm in names:
        H.time_kernel(nm, reps=1)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("probed", names)


if __name__ == "__main__":
    main()
