"""Multi-process (world_size 2, gloo, CPU) tests of the row-slab distributed
solve (tests/slab_dist.py, a test restatement): partition + halo exchange + sharded
MGR V-cycle + distributed GMRES against the single-process oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _mfd_slab_starts(nx, ny, nz):
    slab = nx * ny + (nx + 1) * ny + nx * (ny + 1) + nx * ny
    return [k * slab for k in range(nz)]


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import sys
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, root)
        sys.path.insert(0, os.path.join(root, "tests"))
        import json
        import paper_2101_11649_b200 as mx
        import slab_dist as D
        import refcpu

        nx, ny, nz = 6, 5, 8
        P = mx.mfd_problem(nx, ny, nz, "iid")
        text = mx.load_strategy("mfd_mgr_pi_c1_l1j")
        R = refcpu.RefHierarchy(P.ptr, P.col, P.val, P.partition.field_order, P.partition.labels, text)
        comm = D.Comm()
        be = D.NumpyBackend()
        rr = D.slab_ranges(P.n, _mfd_slab_starts(nx, ny, nz), world)
        a, b = rr[rank]
        A = D.DistOperator(comm, be, (P.ptr, P.col, P.val), rr, rr)
        # distributed SpMV == global (bitwise: same per-row order)
        x = np.random.default_rng(1).standard_normal(P.n)
        y = A.apply(be.vec(x[a:b])).numpy()
        y_ref = refcpu.spmv(P.ptr, P.col, P.val, x)
        spmv_ok = bool(np.array_equal(y, y_ref[a:b]))
        # sharded MGR apply vs the oracle's global apply
        M = D.DistMgr(comm, be, R.dump, R.info(), json.loads(text), rr)
        v = np.random.default_rng(2).uniform(-1, 1, P.n)
        z = M.apply(be.vec(v[a:b])).numpy()
        zr = R.apply(v)[a:b]
        apply_err = float(np.linalg.norm(z - zr) / np.linalg.norm(zr))
        # distributed GMRES
        xs, rep = D.gmres(comm, be, A, M.apply, be.vec(P.rhs[a:b]), be.zeros(b - a), restart=30,
                          rel_tol=1e-6)
        _, rrep = R.solve(P.rhs, restart=30, rel_tol=1e-6)
        q.put((rank, spmv_ok, apply_err, rep["converged"], rep["iterations"], rrep["iterations"],
               rep["history"][:5], rrep["history"][:5], len(A.plan.halo_global)))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, "error", traceback.format_exc()))


@pytest.mark.parametrize("world", [2])
def test_sharded_mgr_gmres_matches_oracle(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
    for r in res:
        assert r[1] != "error", r[2]
        rank, spmv_ok, apply_err, conv, its, rits, h, hr, nhalo = r
        assert spmv_ok
        assert nhalo > 0  # the slabs really exchange a halo
        assert apply_err <= 1e-12, apply_err
        assert conv and abs(its - rits) <= 1
        assert np.allclose(h, hr, rtol=1e-8, atol=1e-10)


def test_slab_ranges_are_contiguous_and_cover():
    import slab_dist as D
    starts = [0, 10, 20, 30, 40, 50, 60, 70]
    for w in (1, 2, 4, 8):
        rr = D.slab_ranges(80, starts, w)
        assert rr[0][0] == 0 and rr[-1][1] == 80
        assert all(rr[i][1] == rr[i + 1][0] for i in range(w - 1))
    flags = np.array([1, 0, 1, 1, 0, 0, 1, 0], bool)
    assert D.ranges_from_flags(flags, [(0, 4), (4, 8)]) == [(0, 3), (3, 4)]


def _transport_worker(rank, world, port, q):
    """The gloo closures behind mx.TransportGroup.torch_distributed (the
    host-transport group of the multi-process sharded path), without a GPU:
    the group object itself needs none, only Shard creation does."""
    try:
        import os
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
        import torch.distributed as dist
        import paper_2101_11649_b200 as mx
        dist.init_process_group("gloo", rank=rank, world_size=world)
        seen = {}
        real = mx.TransportGroup.__init__

        def spy(self, size, exchange, allgather):
            seen["exchange"], seen["allgather"] = exchange, allgather
            real(self, size, exchange, allgather)  # the C-ABI group object (no device needed)

        mx.TransportGroup.__init__ = spy
        g = mx.TransportGroup.torch_distributed()
        peer = 1 - rank
        a, b = np.full(5, float(rank)), np.empty(5)
        seen["exchange"]([(peer, a)], [(peer, b)])
        dst = np.empty(3 * world)
        seen["allgather"](np.array([rank, rank + 0.5, rank + 0.25]), dst)
        # a one-sided call (scatter setup: rank 0 only sends, the others only receive)
        c = np.empty(4)
        if rank == 0:
            seen["exchange"]([(1, np.arange(4.0))], [])
        else:
            seen["exchange"]([], [(0, c)])
        g.close()
        q.put((rank, b.tolist(), dst.tolist(), c.tolist() if rank else None, g.size))
        dist.destroy_process_group()
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, "error", traceback.format_exc()))


def test_host_transport_group_over_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_transport_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in ps:
        p.join(timeout=60)
    for r in res:
        assert r[1] != "error", r[2]
        rank, b, dst, c, size = r
        assert size == 2
        assert b == [float(1 - rank)] * 5
        assert dst == [0.0, 0.5, 0.25, 1.0, 1.5, 1.25]
        if rank:
            assert c == [0.0, 1.0, 2.0, 3.0]
