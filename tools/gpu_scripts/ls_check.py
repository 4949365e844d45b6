"""Quick GPU check of the low-sync (cgs2) GMRES vs MGS: histories, iterations, time."""
import sys, time, os
import numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2101_11649_b200 as mx, refcpu

def run(P, strat, rtol, reps=3):
    t = mx.load_strategy(strat)
    H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, t, P.unknown_map)
    out = {}
    for o in ("mgs", "cgs2"):
        cfg = mx.KrylovConfig(restart=30, rel_tol=rtol, ortho=o)
        x, rep = H.solve(P.rhs, None, cfg)
        ts = []
        for _ in range(reps):
            _, r2 = H.solve(P.rhs, None, cfg)
            ts.append(r2.solve_s)
        out[o] = (rep, min(ts), x)
    hm, hc = np.array(out["mgs"][0].residual_history[:10]), np.array(out["cgs2"][0].residual_history[:10])
    rel = np.max(np.abs(hm - hc) / np.maximum(hm, hm[0]))
    print(f"{strat} n={P.n} its mgs={out['mgs'][0].iterations} cgs2={out['cgs2'][0].iterations} "
          f"t mgs={out['mgs'][1]*1e3:.2f}ms cgs2={out['cgs2'][1]*1e3:.2f}ms hist_rel={rel:.2e} "
          f"launches={out['cgs2'][0].gpu_launches}", flush=True)
    return H

P = mx.mfd_problem(20, 20, 10, "iid"); run(P, "mfd_mgr_pi_c1_l1j", 1e-6)
P = mx.frac_problem(12); run(P, "frac_mgr_u_l1j", 1e-6)
P = mx.mfd_problem(128, 128, 64, "layered", sigma=1.5, seed=20210129)
H = run(P, "mfd_mgr_pi_c1_l1j", 1e-6)
for k in (0, 3, 8, 15, 29):
    for w in ("cgs2", "cgs2dots", "cgs2upd"):
        ms, by = H.time_kernel(f"{w}.{k}", reps=20)
        print(f"  {w}.{k}: {ms*1e3:.1f} us {by/ms/1e6:.0f} GB/s", flush=True)
    if k in (3, 15, 29):
        try:
            ms, by = H.time_kernel(f"arnoldi.{k}", reps=20)
            print(f"  arnoldi.{k}: {ms*1e3:.1f} us {by/ms/1e6:.0f} GB/s", flush=True)
        except Exception as e:
            print(e)
P = mx.comp_problem(100, 100, 50, wells=8, seed=20210130); run(P, "comp_mgr_l1j", 1e-5)
P = mx.frac_problem(64, seed=20210131); run(P, "frac_mgr_u_l1j", 1e-6)
P = mx.comp_problem(128, 128, 64, wells=16, seed=20210134); run(P, "comp_mgr_l1j", 1e-5)
