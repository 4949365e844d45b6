"""GS variant timing at cfg2 (mfd_mgr_pi_c1: 1 V-cycle, hybrid GS) and per-level sweep probes."""
import os, sys, time
sys.path.insert(0, '.')
import paper_2101_11649_b200 as mx
P = mx.mfd_problem(128, 128, 64, "layered", sigma=1.5, seed=20210129)
for strat in sys.argv[1:] or ["mfd_mgr_pi_c1"]:
    H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, mx.load_strategy(strat))
    cfg = mx.KrylovConfig(restart=30, rel_tol=1e-6)
    _, r = H.solve(P.rhs, None, cfg)
    ts = []
    for _ in range(2):
        _, r = H.solve(P.rhs, None, cfg)
        ts.append(r.solve_s)
    print(f"{strat} blk_rows={os.environ.get('MGRX_GS_BLK_ROWS', 'default')} its={r.iterations} solve={min(ts)*1e3:.1f} ms", flush=True)
    info = H.info()
    for k in range(info["coarse_amg_levels"] - 1):
        out = []
        for w in ("pre", "post"):
            ms, by = H.time_kernel(f"amg.{k}.{w}", reps=5)
            out.append(f"{w} {ms*1e3:.1f}us")
        print(f"  amg.{k}: " + " ".join(out), flush=True)
