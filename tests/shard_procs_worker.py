"""Worker of tests/test_gpu_shard_procs.py: one RANK of a torchrun launch
(gloo), every rank a separate process driving the same GPU through libmgrx's
host-transport group (mgrx_transport_group_create). Rank 0 holds the global
hierarchy (scattered setup) or every rank builds its replica; results go to
rank 0, which compares them with the single-GPU path."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.join(HERE, "golden"))
import paper_2101_11649_b200 as mx  # noqa: E402
from test_gpu_shard import _problem  # noqa: E402


def main():
    kind, setup = sys.argv[1], sys.argv[2]
    dist.init_process_group("gloo")
    rank, size = dist.get_rank(), dist.get_world_size()
    os.environ["LOCAL_RANK"] = "0"  # every rank drives the one GPU (mx.default_context reads LOCAL_RANK)
    torch.cuda.set_device(0)
    P, text, rtol = _problem(kind)
    starts = mx.slab_row_starts(P, size)
    g = mx.TransportGroup.torch_distributed()
    H = None
    if setup == "replicated" or rank == 0:
        H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, text, P.unknown_map)
    if setup == "scatter":
        S = mx.Shard(H, rank, size, starts, group=g, scatter=True, ctx=None if H is not None else mx.default_context())
    else:
        S = mx.Shard(H, rank, size, starts, group=g)
    assert S.row_begin == starts[rank] and S.row_end == starts[rank + 1]
    assert not S.fused
    v = np.random.default_rng(7).uniform(-1, 1, P.n)
    out = {"rows": (S.row_begin, S.row_end), "z": S.apply(v[S.row_begin:S.row_end])}
    for o in ("mgs", "cgs2"):
        x, rep = S.solve(P.rhs[S.row_begin:S.row_end], None, mx.KrylovConfig(restart=30, rel_tol=rtol, ortho=o))
        out[o] = (x, rep.converged, rep.iterations, rep.residual_history)
    gathered = [None] * size if rank == 0 else None
    dist.gather_object(out, gathered, dst=0)
    if rank == 0:
        z = H.apply(v)
        for q in gathered:
            b, e = q["rows"]
            assert np.array_equal(q["z"].view(np.int64), z[b:e].view(np.int64)), (kind, b)
        import scipy.sparse as sp
        M = sp.csr_matrix((P.val, P.col, P.ptr), shape=(P.n, P.n))
        for o in ("mgs", "cgs2"):
            assert all(q[o][1] for q in gathered)
            assert all(q[o][3] == gathered[0][o][3] for q in gathered), o
            _, r1 = H.solve(P.rhs, None, mx.KrylovConfig(restart=30, rel_tol=rtol, ortho=o))
            assert abs(gathered[0][o][2] - r1.iterations) <= 1, (o, gathered[0][o][2], r1.iterations)
            k = min(10, len(r1.residual_history), len(gathered[0][o][3]))
            h, hr = np.array(gathered[0][o][3][:k]), np.array(r1.residual_history[:k])
            assert np.all(np.abs(h - hr) <= 1e-10 * np.maximum(np.abs(hr), 1.0)), (o, h, hr)
            x = np.concatenate([q[o][0] for q in gathered])
            assert np.linalg.norm(P.rhs - M @ x) <= rtol * np.linalg.norm(P.rhs) * (1 + 1e-9)
        print("ok", kind, setup, size, gathered[0]["mgs"][2], gathered[0]["cgs2"][2], flush=True)
    dist.barrier()
    S.close()
    g.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
