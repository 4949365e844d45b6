"""Row-slab sharded solve through the C ABI: ranks run as
threads of one process on one GPU (a "local group": halo exchanges and
all-gathers are device copies ordered by events and host barriers; the NCCL
path swaps in ncclSend/ncclRecv/ncclAllGather behind the same two calls).

Bars: the sharded preconditioner application equals the owned rows of the
single-GPU application bit for bit (same rows, same entry order, same
arithmetic); every rank reports the same residual history (partials summed
in rank order); against the single-GPU solve: iterations within +-1 and the
history within 1e-10 relative (only the inner-product reduction order
differs); the assembled solution meets rtol.
"""
import json
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import scipy.sparse as sp

import make_golden
import paper_2101_11649_b200 as mx

pytestmark = pytest.mark.gpu


def _problem(kind):
    if kind == "mfd":
        P = mx.mfd_problem(12, 12, 8, "layered")
        return P, mx.load_strategy("mfd_mgr_pi_c1_l1j"), 1e-6
    if kind == "comp":
        P = mx.comp_problem(10, 10, 6, wells=2)
        return P, mx.load_strategy("comp_mgr_l1j"), 1e-5
    if kind == "frac":
        P = mx.frac_problem(8)
        return P, mx.load_strategy("frac_mgr_u_l1j"), 1e-6
    if kind == "global_relax":
        ptr, col, val, fields, labels, um, rhs = make_golden.build_problem({"kind": "sdd2", "n": 200})
        P = mx.Problem(ptr, col, val, rhs, mx.DofPartition(fields, labels), um, {})
        return P, json.dumps(make_golden.GLOBAL_RELAX), 1e-9
    if kind == "amg_cycles":
        P = mx.mfd_problem(10, 9, 6, "iid")
        s = json.loads(mx.load_strategy("mfd_mgr_pi_c1_l1j"))
        s["coarse"]["cycles"] = 3
        s["levels"][0]["f_relax"] = {"kind": "l1_jacobi", "sweeps": 3, "weight": 0.9}
        return P, json.dumps(s), 1e-7
    raise ValueError(kind)


def _run(shards, fn):
    with ThreadPoolExecutor(len(shards)) as ex:
        return list(ex.map(fn, shards))


@pytest.mark.parametrize("size", [2, 3])
@pytest.mark.parametrize("kind", ["mfd", "comp", "frac", "global_relax", "amg_cycles"])
def test_sharded_apply_and_solve(kind, size):
    P, text, rtol = _problem(kind)
    H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, text, P.unknown_map)
    g = mx.LocalGroup(size)
    starts = mx.slab_row_starts(P, size)
    shards = [mx.Shard(H, r, size, starts, group=g) for r in range(size)]
    assert [s.row_begin for s in shards] == list(starts[:-1])
    v = np.random.default_rng(7).uniform(-1, 1, P.n)
    z = H.apply(v)
    zs = _run(shards, lambda s: s.apply(v[s.row_begin:s.row_end]))
    for s, zr in zip(shards, zs):
        assert np.array_equal(zr.view(np.int64), z[s.row_begin:s.row_end].view(np.int64)), (kind, s.row_begin)
    cfg = mx.KrylovConfig(restart=30, rel_tol=rtol, ortho="mgs")
    x1, r1 = H.solve(P.rhs, None, cfg)
    outs = _run(shards, lambda s: s.solve(P.rhs[s.row_begin:s.row_end], None, cfg))
    reps = [o[1] for o in outs]
    assert all(r.converged for r in reps)
    assert all(r.residual_history == reps[0].residual_history for r in reps)
    assert abs(reps[0].iterations - r1.iterations) <= 1
    k = min(10, len(r1.residual_history), len(reps[0].residual_history))
    h, hr = np.array(reps[0].residual_history[:k]), np.array(r1.residual_history[:k])
    assert np.all(np.abs(h - hr) <= 1e-10 * np.maximum(np.abs(hr), np.abs(hr[0]))), (h, hr)
    x = np.concatenate([o[0] for o in outs])
    M = sp.csr_matrix((P.val, P.col, P.ptr), shape=(P.n, P.n))
    assert np.linalg.norm(P.rhs - M @ x) <= rtol * np.linalg.norm(P.rhs) * (1 + 1e-9)
    for s in shards:
        s.close()
    g.close()


@pytest.mark.parametrize("size", [1, 2, 3])
@pytest.mark.parametrize("kind", ["mfd", "comp", "frac", "amg_cycles"])
def test_sharded_lowsync_solve(kind, size):
    """The default low-synchronisation GMRES on the slabs (two all-gathered
    reductions per step): every rank reports the same history; against the
    single-GPU low-sync solve and the single-GPU MGS solve the north_star bar
    holds (history 1e-10 of the initial residual, iterations +-1) and the
    assembled solution meets rtol."""
    P, text, rtol = _problem(kind)
    H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, text, P.unknown_map)
    g = mx.LocalGroup(size)
    starts = mx.slab_row_starts(P, size)
    shards = [mx.Shard(H, r, size, starts, group=g) for r in range(size)]
    cfg = mx.KrylovConfig(restart=30, rel_tol=rtol, ortho="cgs2")
    outs = _run(shards, lambda s: s.solve(P.rhs[s.row_begin:s.row_end], None, cfg))
    reps = [o[1] for o in outs]
    assert all(r.converged for r in reps)
    assert all(r.residual_history == reps[0].residual_history for r in reps)
    for o in ("cgs2", "mgs"):
        _, r1 = H.solve(P.rhs, None, mx.KrylovConfig(restart=30, rel_tol=rtol, ortho=o))
        assert abs(reps[0].iterations - r1.iterations) <= 1, (o, reps[0].iterations, r1.iterations)
        k = min(10, len(r1.residual_history), len(reps[0].residual_history))
        h, hr = np.array(reps[0].residual_history[:k]), np.array(r1.residual_history[:k])
        assert np.all(np.abs(h - hr) <= 1e-10 * np.maximum(np.abs(hr), 1.0)), (o, h, hr)
    x = np.concatenate([o[0] for o in outs])
    M = sp.csr_matrix((P.val, P.col, P.ptr), shape=(P.n, P.n))
    assert np.linalg.norm(P.rhs - M @ x) <= rtol * np.linalg.norm(P.rhs) * (1 + 1e-9)
    for s in shards:
        s.close()
    g.close()


@pytest.mark.parametrize("size", [2, 3])
@pytest.mark.parametrize("kind", ["mfd", "comp", "frac", "global_relax", "amg_cycles"])
def test_scatter_setup_equals_replicated(kind, size):
    """mgrx_shard_create_scatter (build on rank 0, scatter):
    only rank 0 holds the global hierarchy; the other ranks receive their
    slab plans and rebuild the small replicated parts themselves. The
    shards apply the preconditioner bitwise like the single GPU, solve
    bitwise like the replicated-setup shards (MGS and low-sync), and keep
    working after rank 0 drops the global hierarchy."""
    import gc
    P, text, rtol = _problem(kind)
    H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, text, P.unknown_map)
    starts = mx.slab_row_starts(P, size)
    v = np.random.default_rng(7).uniform(-1, 1, P.n)
    z = H.apply(v)
    g = mx.LocalGroup(size)
    shards = _run(list(range(size)), lambda r: mx.Shard(H if r == 0 else None, r, size, starts, group=g,
                                                        scatter=True, ctx=H.ctx))
    gr = mx.LocalGroup(size)
    repl = [mx.Shard(H, r, size, starts, group=gr) for r in range(size)]
    assert [s.row_begin for s in shards] == list(starts[:-1])
    # each rank's footprint is its slab (plus small replicated coarse parts)
    assert all(s.device_bytes() > 0 for s in shards)
    if kind in ("mfd", "comp", "frac"):
        assert all(s.device_bytes() < H.device_bytes() for s in shards), [s.device_bytes() for s in shards]
    zs = _run(shards, lambda s: s.apply(v[s.row_begin:s.row_end]))
    for s, zr in zip(shards, zs):
        assert np.array_equal(zr.view(np.int64), z[s.row_begin:s.row_end].view(np.int64)), (kind, s.row_begin)
    del H
    gc.collect()
    for o in ("mgs", "cgs2"):
        cfg = mx.KrylovConfig(restart=30, rel_tol=rtol, ortho=o)
        a = _run(shards, lambda s: s.solve(P.rhs[s.row_begin:s.row_end], None, cfg))
        b = _run(repl, lambda s: s.solve(P.rhs[s.row_begin:s.row_end], None, cfg))
        assert all(x[1].converged for x in a)
        assert a[0][1].residual_history == b[0][1].residual_history, o
        xa, xb = np.concatenate([x[0] for x in a]), np.concatenate([x[0] for x in b])
        assert np.array_equal(xa.view(np.int64), xb.view(np.int64)), o
    for s in shards + repl:
        s.close()
    g.close()
    gr.close()


def test_scatter_setup_errors_reach_every_rank():
    """A strategy the slabs cannot run (one-range hybrid Gauss-Seidel) fails
    on rank 0's planner; every rank gets the message instead of waiting."""
    P = mx.mfd_problem(6, 5, 4, "iid")
    H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, mx.load_strategy("mfd_mgr_pi_c1"))
    g = mx.LocalGroup(2)
    st = mx.slab_row_starts(P, 2)

    def mk(r):
        try:
            mx.Shard(H if r == 0 else None, r, 2, st, group=g, scatter=True, ctx=H.ctx)
        except mx.MgrxError as e:
            return str(e)
        return "no error"
    msgs = _run([0, 1], mk)
    assert all("hybrid Gauss-Seidel is a sequential sweep" in m for m in msgs), msgs
    with pytest.raises(mx.MgrxInvalidArgument, match="rank 0"):
        mx.Shard(None, 0, 1, [0, P.n], scatter=True, ctx=H.ctx)


def test_sharded_rejects_sequential_gs():
    P = mx.mfd_problem(6, 5, 4, "iid")
    H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, mx.load_strategy("mfd_mgr_pi_c1"))
    g = mx.LocalGroup(2)
    with pytest.raises(mx.MgrxError, match="hybrid Gauss-Seidel is a sequential sweep"):
        mx.Shard(H, 0, 2, None, group=g)
    with pytest.raises(mx.MgrxInvalidArgument, match="row starts"):
        mx.Shard(H, 0, 2, [0, 5, P.n - 1], group=g)


def test_single_rank_shard_equals_global():
    """size 1: the sharded code path (no exchanges) reproduces the global
    solve bit for bit, including the inner products (one rank = the
    canonical per-rank order)."""
    P = mx.mfd_problem(12, 10, 6, "iid")
    H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, mx.load_strategy("mfd_mgr_pi_c1_l1j"))
    S = mx.Shard(H, 0, 1)
    cfg = mx.KrylovConfig(restart=30, rel_tol=1e-8, ortho="mgs")
    x1, r1 = H.solve(P.rhs, None, cfg)
    x2, r2 = S.solve(P.rhs, None, cfg)
    assert r2.residual_history == r1.residual_history
    assert np.array_equal(x2.view(np.int64), x1.view(np.int64))


def test_nccl_single_rank():
    """The NCCL communicator (libnccl dlopen'ed, ncclCommInitRank, the
    all-gathered inner products) on one rank reproduces the global solve."""
    P = mx.mfd_problem(10, 10, 5, "iid")
    H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, mx.load_strategy("mfd_mgr_pi_c1_l1j"))
    S = mx.Shard(H, 0, 1, None, nccl_id=mx.nccl_unique_id())
    cfg = mx.KrylovConfig(restart=30, rel_tol=1e-8, ortho="mgs")
    x1, r1 = H.solve(P.rhs, None, cfg)
    x2, r2 = S.solve(P.rhs, None, cfg)
    assert r2.residual_history == r1.residual_history
    assert np.array_equal(x2.view(np.int64), x1.view(np.int64))
    S.close()


def test_sharded_without_replicated_coarse_levels():
    """MGRX_SHARD_REPL_ROWS=0 keeps every AMG level sharded (halo exchanges
    down to the coarsest); the default replicates the levels of <= 64K rows
    (one all-gather, then the single-GPU kernels). Both are bitwise equal to
    the single-GPU application."""
    import os
    import subprocess
    import sys
    code = (
        "import sys, numpy as np; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')\n"
        "from concurrent.futures import ThreadPoolExecutor\n"
        "import paper_2101_11649_b200 as mx\n"
        "for size in (2, 3):\n"
        "    P = mx.mfd_problem(12, 12, 8, 'layered')\n"
        "    H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, mx.load_strategy('mfd_mgr_pi_c1_l1j'))\n"
        "    g = mx.LocalGroup(size); st = mx.slab_row_starts(P, size)\n"
        "    S = [mx.Shard(H, r, size, st, group=g) for r in range(size)]\n"
        "    v = np.random.default_rng(7).uniform(-1, 1, P.n); z = H.apply(v)\n"
        "    with ThreadPoolExecutor(size) as ex: zs = list(ex.map(lambda s: s.apply(v[s.row_begin:s.row_end]), S))\n"
        "    for s, zr in zip(S, zs): assert np.array_equal(zr.view(np.int64), z[s.row_begin:s.row_end].view(np.int64))\n"
        "    [s.close() for s in S]; g.close()\n"
        "print('ok')")
    root = make_golden.ROOT
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                         env={**os.environ, "MGRX_SHARD_REPL_ROWS": "0"}, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]
