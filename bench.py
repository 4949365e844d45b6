"""Benchmark: MGR-preconditioned GMRES on BASELINE cfg2 (hybrid-MFD [p, pi]
system on a 128x128x64 grid with a layered log-normal permeability field,
4,227,072 DOF), FGMRES(30), rtol 1e-6, strategy = one exact reduction of the
face multipliers (ideal interp, injection) + one AMG V-cycle on the cell
pressure system with l1-Jacobi x2 AMG smoothing
(strategies/mfd_mgr_pi_c1_l1j.json: BASELINE cfg2's "one AMG V-cycle"; the
shipped proj/strategies/mfd_mgr_pi.json, 8 V-cycles of hybrid Gauss-Seidel,
is measured in the same line under "variants"). Orthogonalisation: the
default low-synchronisation lagged CGS2 (csrc/lowsync.cu) with the
tolerance-level team-sum SpMV kernels where the setup timing picks them; the
reference's MGS (bitwise parity mode, left-to-right row sums) is a variant.

A step = one complete solve from x0 = 0 with the hierarchy already built
(setup is timed separately and reported). value = DOF * GMRES iterations /
solve time, summed over ranks. Inputs (matrix 200 MB + hierarchy) exceed the
126 MB L2, so no explicit flush is needed between steps.

--impl reference times the reference CPU implementation of the path (the
refcpu oracle: the reference itself cannot be compiled here) on
the host cores, on a bounded sample of the same workload.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MGR-FGMRES DOF*iters/sec"
UNIT = "DOF*iters/s"
# Workloads (BASELINE.json configs). cfg2 is the headline (the metric's
# config, single GPU); the others are available for measurements and parity.
CONFIGS = {
    "cfg1": {"kind": "mfd", "dims": (20, 20, 10), "field": "iid", "seed": 20210128,
             "strategy": "mfd_mgr_pi_c1", "rtol": 1e-6,
             "desc": "cfg1: hybrid-MFD [p,pi] 20x20x10 iid log-normal, FGMRES(30) rtol 1e-6, MGR_pi + 1 AMG V-cycle"},
    "cfg2": {"kind": "mfd", "dims": (128, 128, 64), "field": "layered", "seed": 20210129,
             "strategy": "mfd_mgr_pi_c1_l1j", "rtol": 1e-6, "variant": ["mfd_mgr_pi", "mfd_mgr_pi_c1"],
             "desc": "cfg2: hybrid-MFD [p,pi] 128x128x64 layered log-normal (1e6 contrast), "
                     "FGMRES(30) rtol 1e-6, MGR_pi (exact pi elimination) + 1 AMG V-cycle "
                     "(l1-Jacobi x2 AMG smoothing; variant: the AMG default hybrid Gauss-Seidel)"},
    "cfg3": {"kind": "comp", "dims": (100, 100, 50), "wells": 8, "seed": 20210130,
             "strategy": "comp_mgr_l1j", "rtol": 1e-5, "variant": ["comp_mgr"],
             "desc": "cfg3: compositional p+3 densities 100x100x50 (4x4 blocks) + 8 wells x 50 elements x 5 dofs, "
                     "FGMRES(30) rtol 1e-5, MGR rho3 -> rho1,rho2 -> p(AMG, l1-Jacobi x2; variant: hybrid GS) "
                     "-> wells(dense LU)"},
    "cfg4": {"kind": "frac", "m": 64, "seed": 20210131, "strategy": "frac_mgr_u_l1j", "rtol": 1e-6,
             "variant": ["frac_mgr_u"],
             "desc": "cfg4: 3-D Q1 elasticity 64^3 nodes (81 nnz/row) + mid-plane fracture lubrication, "
                     "FGMRES(30) rtol 1e-6, MGR_u with unknown-based AMG on A_uu (l1-Jacobi x2; variant: "
                     "hybrid GS), AMG coarse on p"},
    # cfg5: cfg3 physics weak-scaled to 1,048,576 cells per GPU (z-slabs),
    # 8 wells per 500k cells; dims for N = 1/2/4/8 GPUs follow SURVEY §8(d).
    "cfg5": {"kind": "comp", "dims_by_n": {1: (128, 128, 64), 2: (128, 128, 128), 4: (256, 128, 128),
                                           8: (256, 256, 128)},
             "seed": 20210134, "strategy": "comp_mgr_l1j", "rtol": 1e-5, "weak": True,
             "desc": "cfg5: cfg3 physics weak-scaled, 1,048,576 cells (4 dofs) per GPU + 8 wells per 500k cells, "
                     "z-slab partition with NCCL halo exchanges, FGMRES(30) rtol 1e-5, comp_mgr_l1j"},
}
CONFIG = "cfg2"
STRATEGY = CONFIGS[CONFIG]["strategy"]
RTOL = CONFIGS[CONFIG]["rtol"]
RESTART = 30


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


class Clocks:
    """nvidia-smi sampling during the timed region."""

    def __init__(self, gpu):
        self.gpu, self.samples, self.proc = gpu, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            p = [x.strip() for x in line.split(",")]
            if len(p) >= 7:
                self.samples.append(p)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        import statistics
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4) if s[3 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def make_problem(n_gpus=1):
    import paper_2101_11649_b200 as mx
    c = CONFIGS[CONFIG]
    if "dims_by_n" in c:
        dims = c["dims_by_n"].get(n_gpus) or (128, 128, 64 * n_gpus)
        cells = dims[0] * dims[1] * dims[2]
        return mx.comp_problem(*dims, wells=max(1, (8 * cells) // 500000), seed=c["seed"])
    if c["kind"] == "mfd":
        return mx.mfd_problem(*c["dims"], c["field"], sigma=1.5, seed=c["seed"])
    if c["kind"] == "frac":
        return mx.frac_problem(c["m"], seed=c["seed"])
    return mx.comp_problem(*c["dims"], wells=c["wells"], seed=c["seed"])


def cpu_reference(P, steps, warmup, max_iters, threads, single_iters=0):
    """refcpu oracle: setup once, then each step = a GMRES solve capped at
    max_iters iterations (bounded sample). Returns DOF*iters/s."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import refcpu
    import paper_2101_11649_b200 as mx
    refcpu.set_threads(threads)
    H = refcpu.RefHierarchy(P.ptr, P.col, P.val, P.partition.field_order, P.partition.labels,
                            mx.load_strategy(STRATEGY), P.unknown_map)
    for _ in range(warmup):
        H.solve(P.rhs, restart=RESTART, max_iters=max_iters, rel_tol=RTOL)
    its, t = 0, 0.0
    for _ in range(steps):
        t0 = time.perf_counter()
        _, rep = H.solve(P.rhs, restart=RESTART, max_iters=max_iters, rel_tol=RTOL)
        t += time.perf_counter() - t0
        its += rep["iterations"]
    single = None
    if single_iters:
        # the faithful single-threaded reference (same hierarchy)
        refcpu.set_threads(1)
        t0 = time.perf_counter()
        _, rep = H.solve(P.rhs, restart=RESTART, max_iters=single_iters, rel_tol=RTOL)
        ts = time.perf_counter() - t0
        single = {"value": P.n * rep["iterations"] / ts, "cores": 1,
                  "sample": f"one solve capped at {rep['iterations']} iterations ({ts:.1f}s)"}
        refcpu.set_threads(threads)
    return P.n * its / t, t, its, H.setup_s, single


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    P = make_problem(world)
    threads = os.cpu_count() or 1
    v, t, its, setup_s, _ = cpu_reference(P, args.steps, args.warmup, args.ref_iters, threads)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / max(args.steps, 1),
            "higher_is_better": True, "scaling": scaling_kind(world), "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(P, args.gpus),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"{CONFIG} MGR-GMRES solves capped at {args.ref_iters} iterations "
                                       f"({its} iterations over {args.steps} steps), setup {setup_s:.1f}s excluded"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def scaling_kind(n_gpus):
    """cfg5 fixes the work per GPU; the other configs split one problem."""
    return "weak" if (CONFIGS[CONFIG].get("weak") or n_gpus == 1) else "strong"


STRATEGY_NOTES = {
    "mfd_mgr_pi_c1_l1j": "BASELINE cfg2 fixes one exact reduction + ONE AMG V-cycle but not the AMG smoother; "
                         "this strategy file (reference JSON schema) uses l1-Jacobi x2, the north_star's "
                         "relaxation family. The shipped proj/strategies/mfd_mgr_pi.json (8 V-cycles, hybrid "
                         "Gauss-Seidel) and its 1-cycle form are timed under variants.",
    "comp_mgr_l1j": "l1-Jacobi x2 AMG smoothing in the reference schema; the shipped-style comp_mgr "
                    "(hybrid Gauss-Seidel) is timed under variants.",
    "frac_mgr_u_l1j": "l1-Jacobi x2 AMG smoothing in the reference schema; the shipped frac_mgr_u (hybrid "
                      "Gauss-Seidel) is timed under variants.",
}


def workload_config(P, n_gpus):
    return {"workload": CONFIGS[CONFIG]["desc"],
            "dofs": int(P.n), "nnz": int(P.ptr[-1]), "strategy": STRATEGY, "restart": RESTART,
            "rel_tol": RTOL, "strategy_note": STRATEGY_NOTES.get(STRATEGY),
            "ortho": "cgs2 (lagged CGS2, 2 basis sweeps + 2 reductions per step, device-resident restart cycle); "
                     "history within the north_star bar of the oracle (tests/test_gpu_fullsize.py)",
            "parallelism": f"zslab{n_gpus} (NCCL halo exchange + all-gathered inner products)"
            if n_gpus > 1 else "single",
            "l2_flush": "inputs exceed L2 (matrix+hierarchy > 126 MB)"}


def probe_names(H):
    info = H.info()
    names = ["cgs2.15", "cgs2dots.15", "cgs2upd.15", "arnoldi.15", "spmv.A", "precond.inexact"]
    if info["mgr_levels"]:
        names += ["mgr.0.rres", "mgr.0.prolong"]
    for k in range(max(info["coarse_amg_levels"] - 1, 0)):
        names += [f"amg.{k}.resid", f"amg.{k}.pre", f"amg.{k}.post"]
    # F-relaxation AMG hierarchies (cfg4: the unknown-based AMG on A_uu, where the time goes)
    for l, nl in enumerate(info["frelax_amg_levels"]):
        for k in range(min(max(nl - 1, 0), 4)):
            names += [f"mgr.{l}.frelax.amg.{k}.resid", f"mgr.{l}.frelax.amg.{k}.pre"]
    return names


def run_sharded(args):
    """N > 1 (one rank per GPU): rank 0 builds the global hierarchy on its GPU
    and scatters every rank its slab plan (mgrx_shard_create_scatter over
    NCCL); no other rank holds a global operator, and rank 0 drops the
    global hierarchy once the shards exist. gloo carries only the NCCL id
    and the max-over-ranks timing. value = global DOF x iterations / (max
    over ranks of the device-timed solve)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2101_11649_b200 as mx

    rank, world, local = dist_env()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(local)
    P = make_problem(world)  # host bundle (rhs slices, row starts); device setup on rank 0 only
    ctx = mx.Context(local)
    H, setup_wall, solve_model = None, 0.0, None
    if rank == 0:
        A = mx.Matrix(P.ptr, P.col, P.val, ctx=ctx)
        t0 = time.perf_counter()
        H = mx.Hierarchy(A, P.partition, mx.load_strategy(STRATEGY), P.unknown_map)
        setup_wall = time.perf_counter() - t0
        try:
            sys.path.insert(0, os.path.join(ROOT, "tools"))
            from solve_model import SolveModel
            solve_model = SolveModel(H, mx.load_strategy(STRATEGY))
        except Exception as e:
            solve_model = e
        hinfo = H.info()
    obj = [mx.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    starts = mx.slab_row_starts(P, world)
    t0 = time.perf_counter()
    S = mx.Shard(H, rank, world, starts, nccl_id=obj[0], scatter=True, ctx=ctx)
    scatter_wall = time.perf_counter() - t0
    if rank == 0:
        if not isinstance(solve_model, Exception):
            solve_model.H = None  # the model keeps only sizes
        del H, A  # the shards do not reference the global hierarchy
    import gc
    gc.collect()
    lo, hi = S.row_begin, S.row_end
    # NCCL communicator of this rank is up: log it and count the ranks that got there
    print(f"[bench rank {rank}/{world}] NCCL communicator ready on cuda:{local} "
          f"(rows {lo}..{hi}, scattered setup {scatter_wall:.2f}s)", file=sys.stderr, flush=True)
    ready = torch.ones(1)
    dist.all_reduce(ready)
    nccl_ranks = int(ready.item())
    assert nccl_ranks == world, (nccl_ranks, world)
    mem = ctx.memory()
    memt = torch.tensor([float(mem["used"]), float(mem["high"])], dtype=torch.float64)
    mems = [torch.zeros(2, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(mems, memt)
    cfg = mx.KrylovConfig(restart=RESTART, max_iters=500, rel_tol=RTOL)
    dev = torch.device("cuda", local)
    b = torch.from_numpy(np.ascontiguousarray(P.rhs[lo:hi])).to(dev)
    x = torch.zeros(hi - lo, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()

    def step():
        return S.solve_device(b.data_ptr(), x.data_ptr(), cfg, zero_guess=True)

    for _ in range(args.warmup):
        step()
    dist.barrier()
    torch.cuda.synchronize()
    its, launches, dev_s = 0, 0, 0.0
    with Clocks(local) as clk:
        for _ in range(args.steps):
            rep = step()
            its += rep.iterations
            launches += rep.gpu_launches
            dev_s += rep.solve_s  # CUDA events on the shard's stream
        torch.cuda.synchronize()
    dist.barrier()
    t = torch.tensor([dev_s], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_max = float(t.item())
    value = P.n * its / t_max
    # e2e: the public API with pinned host slices (H2D of b, D2H of x)
    b_host = torch.empty(hi - lo, dtype=torch.float64, pin_memory=True).numpy()
    b_host[:] = P.rhs[lo:hi]
    x_host = torch.empty(hi - lo, dtype=torch.float64, pin_memory=True).numpy()
    S.solve(b_host, None, cfg, out=x_host)
    dist.barrier()
    te, e_its = 0.0, 0
    for _ in range(args.steps):
        t1 = time.perf_counter()
        _, rep_e = S.solve(b_host, None, cfg, out=x_host)
        te += time.perf_counter() - t1
        e_its += rep_e.iterations
    tt = torch.tensor([te], dtype=torch.float64)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    e2e = P.n * e_its / float(tt.item())
    nb = torch.tensor([8.0 * (hi - lo)], dtype=torch.float64)
    dist.all_reduce(nb, op=dist.ReduceOp.SUM)
    solve_roof = None
    if rank == 0:
        # whole-job roofline: the single-GPU byte model of the global solve
        # (halo traffic excluded) over N GPUs' HBM for the max-over-ranks time
        try:
            if isinstance(solve_model, Exception):
                raise solve_model
            peak, peak_kind = peaks()
            mb = solve_model.solve_bytes(int(P.ptr[-1]), P.n, int(round(its / args.steps)), RESTART, ortho="cgs2")
            ts = t_max / args.steps
            solve_roof = {"bound": "hbm", "model_bytes_per_solve": mb["bytes"],
                          "achieved": mb["bytes"] / ts / 1e9, "peak": peak * world, "unit": "GB/s",
                          "frac": mb["bytes"] / ts / 1e9 / (peak * world), "peak_source": peak_kind,
                          "model": "tools/solve_model.py (global solve, halo traffic not counted), "
                                   "peak = N x per-GPU HBM"}
        except Exception as e:
            solve_roof = {"error": f"{type(e).__name__}: {e}"}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps, "higher_is_better": True,
                "scaling": scaling_kind(world), "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {**workload_config(P, world), "row_starts": [int(v) for v in starts]},
                "iterations_per_solve": its / args.steps, "solve_time_s": t_max / args.steps,
                "setup_wall_s": setup_wall, "scatter_wall_s": scatter_wall, "hierarchy": hinfo,
                "setup": "rank 0 builds the global hierarchy and scatters slab plans (mgrx_shard_create_scatter); "
                         "no other rank holds a global operator",
                "device_mem_used_bytes_per_rank": [int(m[0].item()) for m in mems],
                "device_mem_high_bytes_per_rank": [int(m[1].item()) for m in mems],
                "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": int(nb.item()),
                        "d2h_bytes_per_step": int(nb.item()),
                        "path": "Shard.solve -> mgrx_shard_solve (C ABI) per rank, pinned host slices"},
                "gpu_launches": launches, "roofline": None, "solve_roofline": solve_roof, "cpu_baseline": None,
                "fused_sharded_arnoldi": bool(getattr(S, "fused", False)), "nccl_ranks": nccl_ranks,
                "clocks": clk.summary()}
        print(json.dumps(line))
    S.close()
    dist.barrier()
    dist.destroy_process_group()


def spawn_ranks(args):
    """`python bench.py --gpus N` without a launcher: start N ranks (one per
    GPU) through torch.distributed.run on 127.0.0.1 and pass rank 0's line
    through. Fails loudly when fewer than N GPUs are visible."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} requested but {have} CUDA device(s) visible")
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    rc = subprocess.call(cmd)
    if rc:
        raise SystemExit(rc)


def main():
    global STRATEGY, CONFIG, RTOL
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mgrx")
    ap.add_argument("--ref-iters", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-variant", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="use the z-slab sharded solve even at N=1 (exercises the NCCL path on one GPU)")
    ap.add_argument("--strategy", default=None, help="strategies/<name>.json (default: %s)" % STRATEGY)
    args = ap.parse_args()
    CONFIG = args.config
    STRATEGY = CONFIGS[CONFIG]["strategy"]
    RTOL = CONFIGS[CONFIG]["rtol"]
    if args.strategy:
        STRATEGY = args.strategy
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']}")

    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2101_11649_b200 as mx

    rank, world, local = dist_env()
    if world > 1 or args.sharded:
        return run_sharded(args)
    torch.cuda.set_device(local)
    P = make_problem()
    ctx = mx.Context(local)
    A = mx.Matrix(P.ptr, P.col, P.val, ctx=ctx)
    t0 = time.perf_counter()
    H = mx.Hierarchy(A, P.partition, mx.load_strategy(STRATEGY), P.unknown_map)
    setup_wall = time.perf_counter() - t0
    cfg = mx.KrylovConfig(restart=RESTART, max_iters=500, rel_tol=RTOL)

    dev = torch.device("cuda", local)
    b = torch.from_numpy(P.rhs).to(dev)
    x = torch.zeros(P.n, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()

    def step():
        x.zero_()
        torch.cuda.synchronize()
        return H.solve_device(b.data_ptr(), x.data_ptr(), cfg)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    its, launches, solve_dev = 0, 0, 0.0
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    prof = bool(os.environ.get("MGRX_PROFILE_TIMED"))
    with Clocks(local) as clk:
        if prof:
            torch.cuda.profiler.start()
        start.record()
        for _ in range(args.steps):
            rep = step()
            its += rep.iterations
            launches += rep.gpu_launches
            solve_dev += rep.solve_s
        end.record()
        torch.cuda.synchronize()
        if prof:
            torch.cuda.profiler.stop()
    ms = start.elapsed_time(end)
    value = P.n * its / (ms * 1e-3)

    # e2e: public API with pinned host buffers: H2D of b, zero initial guess
    # (set on the device), D2H of x, all inside the timed region (host clock)
    b_host = torch.empty(P.n, dtype=torch.float64, pin_memory=True).numpy()
    b_host[:] = P.rhs
    x_host = torch.empty(P.n, dtype=torch.float64, pin_memory=True).numpy()
    H.solve(b_host, None, cfg, out=x_host)
    te, e_its = 0.0, 0
    for _ in range(args.steps):
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        _, rep_e = H.solve(b_host, None, cfg, out=x_host)
        te += time.perf_counter() - t1
        e_its += rep_e.iterations
    e2e = P.n * e_its / te

    # roofline: dominant kernel probes (device events on the library stream)
    peak, peak_kind = peaks()
    info = H.info()
    probes = {}
    for name in probe_names(H):
        try:
            ms_k, by = H.time_kernel(name, reps=20)
            probes[name] = {"avg_ms": ms_k, "bytes": by, "GBps": by / (ms_k * 1e-3) / 1e9}
            if by == 0.0:
                del probes[name]["GBps"]  # the whole-application probe: bytes from the solve model below
        except mx.MgrxError as e:
            probes[name] = {"error": str(e)}
    # roofline object: the dominant kernel by time share of one timed solve.
    # profiles/r02/launch_shares_cfg2.txt: k_spmv_xtile 27.8% + k_spmv_staged
    # 19.0% (the staged SpMV and its x-window form, one code family: 1,141
    # launches on the fine operator, the MGR restricted residual and the AMG
    # levels 0-2), k_ls_update 13.4%, k_ls_dots 12.5% (73 launches each); the
    # family also leads cfg3-5. The headline fraction is the family's,
    # time-weighted over every instance of one preconditioner application +
    # the GMRES SpMV (algorithmic bytes summed / launch durations summed),
    # each launch timed from a COLD L2 ("cold:" probes: in a solve ~1.5 GB
    # stream through the 126 MB L2 between two uses of an operator; back-to-
    # back launches of one kernel would re-read sub-L2 working sets from L2).
    # The largest instance (spmv.A, the fine operator) and the two low-sync
    # Arnoldi sweeps at the mean Krylov index (k = 15) are reported beside
    # it. Other strategies: the probe with the largest time.
    share = {k: v["avg_ms"] for k, v in probes.items() if "avg_ms" in v and "GBps" in v}
    if "l1j" in STRATEGY and "avg_ms" in probes.get("spmv.A", {}):
        dom = "spmv.A"
    else:
        dom = max((k for k in share), key=lambda k: share[k])
    d = probes[dom]
    traffic, shares, captured = None, None, {}
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "roofline_traffic.json")) as f:
            tr = json.load(f).get(CONFIG, {})
        traffic = tr.get("kernels", {}).get(dom, {}).get("dram_bytes_per_launch")
        shares = tr.get("launch_shares")
        # ncu DRAM bytes over algorithmic bytes of every captured probe launch
        captured = {k: round(v["traffic_over_algorithmic"], 3) for k, v in tr.get("kernels", {}).items()
                    if isinstance(v, dict) and v.get("traffic_over_algorithmic") is not None}
    except Exception:
        pass
    arn = {}
    for nm, kern in (("cgs2dots.15", "k_ls_dots"), ("cgs2upd.15", "k_ls_update"), ("cgs2.15", "both sweeps")):
        if "avg_ms" in probes.get(nm, {}):
            arn[kern] = {"probe": nm, "achieved": probes[nm]["GBps"], "frac": probes[nm]["GBps"] / peak,
                         "algorithmic_bytes": probes[nm]["bytes"], "avg_ms": probes[nm]["avg_ms"]}
    # the SpMV family as a whole (k_spmv_staged and its x-window form
    # k_spmv_xtile, the team-sum kernels): every probe of a product / sweep /
    # residual on an operator large enough not to be launch-bound, bytes and
    # time summed -- the time-weighted fraction of the family, next to its
    # share of a solve's kernel time (ncu launch list, profiles/r02)
    fam = [k for k, v in probes.items() if "GBps" in v and v["avg_ms"] >= 0.006 and
           (k == "spmv.A" or k.endswith(".rres") or ".amg." in k or k.startswith("amg."))]
    family = None
    if fam:
        for k in fam:  # the same launches from a cold L2 (differential timing, no launch latency)
            try:
                ms_c, _ = H.time_kernel("cold:" + k, reps=20)
                probes[k]["cold_ms"] = ms_c
                probes[k]["cold_GBps"] = probes[k]["bytes"] / (ms_c * 1e-3) / 1e9
            except mx.MgrxError as e:
                probes[k]["cold_error"] = str(e)
        fb, ft = sum(probes[k]["bytes"] for k in fam), sum(probes[k]["avg_ms"] for k in fam) * 1e-3
        fshare = None
        if shares:
            fshare = round(sum(v for k, v in shares.items() if k.startswith("k_spmv") and isinstance(v, float)), 4)
        family = {"kernels": "k_spmv_xtile / k_spmv_staged / k_spmv_vec2 / k_spmv_tbsr3 (SpMV family)",
                  "probes": fam, "bytes": fb, "ms": ft * 1e3, "achieved": fb / ft / 1e9, "frac": fb / ft / 1e9 / peak,
                  "l2": "warm (back-to-back launches)", "share_of_solve_kernel_time": fshare}
        if all("cold_ms" in probes[k] for k in fam):
            fc = sum(probes[k]["cold_ms"] for k in fam) * 1e-3
            family["cold"] = {"ms": fc * 1e3, "achieved": fb / fc / 1e9, "frac": fb / fc / 1e9 / peak,
                              "l2": "cold before every launch"}
    if dom == "spmv.A" and family and "cold" in family:
        # headline: the family (top two kernels by share), cold L2, time-weighted
        inst = {"kernel": "k_spmv_staged", "instance": "spmv.A (fine operator; GMRES SpMV)",
                "achieved": d["GBps"], "frac": d["GBps"] / peak, "algorithmic_bytes": d["bytes"], "traffic": traffic,
                "cold_achieved": d.get("cold_GBps"), "cold_frac": d.get("cold_GBps", 0.0) / peak}
        nl = len(fam)
        roof = {"bound": "hbm", "kernel": "k_spmv_xtile + k_spmv_staged (SpMV family: the two largest launch shares)",
                "instance": f"time-weighted over {nl} instances (GMRES SpMV + one preconditioner application), "
                            "cold L2 before every launch",
                "achieved": family["cold"]["achieved"], "peak": peak, "unit": "GB/s",
                "frac": family["cold"]["frac"], "traffic": None,
                "algorithmic_bytes": fb / nl, "launches_averaged": nl,
                "traffic_over_algorithmic": {k: v for k, v in captured.items() if k in fam} or None,
                "largest_instance": inst}
    else:
        roof = {"bound": "hbm", "kernel": "k_spmv_staged" if dom == "spmv.A" else dom,
                "instance": "spmv.A (fine operator; GMRES SpMV)" if dom == "spmv.A" else dom,
                "achieved": d["GBps"], "peak": peak, "unit": "GB/s",
                "frac": d["GBps"] / peak, "traffic": traffic, "algorithmic_bytes": d["bytes"]}
    roof.update({
            "peak_source": peak_kind, "launch_shares": shares, "spmv_family": family, "arnoldi_low_sync": arn,
            "kernels": probes,
            "probe_method": "CUDA events on the library stream over 20 back-to-back launches (inputs in HBM; "
                            "the L2 may retain part of a working set near its 126 MB size); cold_ms: the "
                            "same launch from a cold L2, (20 x [256 MB flush read, launch] - 20 x [flush read]) / 20"})

    # whole-solve roofline: SURVEY §8(d) compulsory-traffic bytes of one solve
    # (tools/solve_model.py, from the hierarchy's sizes) over the timed solve
    try:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        from solve_model import SolveModel
        sm = SolveModel(H, mx.load_strategy(STRATEGY))
        its_solve = int(round(its / args.steps))
        mb = sm.solve_bytes(int(P.ptr[-1]), P.n, its_solve, RESTART, ortho="cgs2")
        t_solve = ms * 1e-3 / args.steps
        solve_roof = {"bound": "hbm", "model_bytes_per_solve": mb["bytes"],
                      "achieved": mb["bytes"] / t_solve / 1e9, "peak": peak, "unit": "GB/s",
                      "frac": mb["bytes"] / t_solve / 1e9 / peak,
                      "precond_bytes_per_apply": mb["precond_bytes_per_apply"],
                      "precond_apply": ({"avg_ms": probes["precond.inexact"]["avg_ms"],
                                         "achieved": mb["precond_bytes_per_apply"] /
                                         (probes["precond.inexact"]["avg_ms"] * 1e-3) / 1e9,
                                         "frac": mb["precond_bytes_per_apply"] /
                                         (probes["precond.inexact"]["avg_ms"] * 1e-3) / 1e9 / peak}
                                        if "avg_ms" in probes.get("precond.inexact", {}) else None),
                      "spmv_bytes": mb["spmv_bytes"], "restart_cycles": mb["restart_cycles"],
                      "model": "SURVEY 8(d) compulsory traffic per operation (tools/solve_model.py); "
                               "low-sync orthogonalisation at 16n(k+3) per step"}
    except Exception as e:  # the model is reporting, never a reason to lose the line
        solve_roof = {"error": f"{type(e).__name__}: {e}"}

    variants = {}

    def time_solves(Hx, cfgx, reps):
        stepx = lambda: (x.zero_(), torch.cuda.synchronize(), Hx.solve_device(b.data_ptr(), x.data_ptr(), cfgx))[2]
        stepx()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        rv = [stepx() for _ in range(reps)]
        ev1.record()
        torch.cuda.synchronize()
        msx = ev0.elapsed_time(ev1) / len(rv)
        itx = sum(r.iterations for r in rv) / len(rv)
        return {"value": P.n * itx / (msx * 1e-3), "unit": UNIT, "ms_per_step": msx, "iterations_per_solve": itx}

    if not args.no_variant:
        # the reference's MGS orthogonalisation (bitwise parity mode), same strategy
        variants["ortho_mgs"] = {**time_solves(H, mx.KrylovConfig(restart=RESTART, max_iters=500, rel_tol=RTOL,
                                                                   ortho="mgs"), max(1, args.steps // 2)),
                                 "strategy": STRATEGY, "ortho": "mgs (reference MGS, bitwise vs the oracle)"}
    vnames = CONFIGS[CONFIG].get("variant") or []
    if not args.strategy and not args.no_variant:
        for vname in vnames:
            Hv = mx.Hierarchy(A, P.partition, mx.load_strategy(vname), P.unknown_map)
            reps = 1 if vname == "mfd_mgr_pi" else max(1, args.steps // 2)
            variants[vname] = {**time_solves(Hv, cfg, reps), "strategy": vname,
                               "smoother": "hybrid_l1_gs (AMG default; exact sequential Gauss-Seidel, sync-free sweep)",
                               "shipped": vname in ("mfd_mgr_pi", "comp_mgr", "frac_mgr_u")}
            if "amg.0.pre" in probe_names(Hv):
                gs_ms, gs_by = Hv.time_kernel("amg.0.pre", reps=5)
                variants[vname]["dominant_kernel"] = {
                    "name": "k_gs (fine coarse-AMG level, forward sweep)", "avg_ms": gs_ms,
                    "achieved_GBps": gs_by / (gs_ms * 1e-3) / 1e9, "frac": gs_by / (gs_ms * 1e-3) / 1e9 / peak,
                    "bound": "latency (dependency chain of the sequential sweep)"}
            del Hv
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        v, t, cits, setup_s, single = cpu_reference(P, 1, 0, args.ref_iters, threads, single_iters=3)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"refcpu oracle, {CONFIG}, one solve capped at {args.ref_iters} iterations "
                         f"({cits} its in {t:.1f}s; setup {setup_s:.1f}s excluded)",
               "single_thread": single}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": scaling_kind(world), "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": workload_config(P, world),
                "iterations_per_solve": its / args.steps, "solve_time_s": ms * 1e-3 / args.steps,
                "setup_s": rep.setup_s, "setup_wall_s": setup_wall,
                "hierarchy": info,
                "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": 8 * P.n,
                        "d2h_bytes_per_step": 8 * P.n,
                        "path": "Hierarchy.solve -> mgrx_solve (C ABI) with pinned host b / x, zero initial guess"},
                "gpu_launches": launches, "roofline": roof, "solve_roofline": solve_roof, "cpu_baseline": cpu,
                "variants": variants,
                "clocks": clk.summary()}
        print(json.dumps(line))


if __name__ == "__main__":
    main()
