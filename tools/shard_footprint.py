"""Per-rank device footprint of the scattered sharded setup (
VERDICT r1 "Next" #2: per-rank device memory at cfg5 N=8 within ~1.3x of
the N=1 footprint).

N=1: the single-GPU hierarchy of cfg5's 1-GPU point (128x128x64 cells, 16
wells, 4.2M DOF): device bytes of mgrx_setup (matrix copy + hierarchy).
N=8: cfg5 at 8 GPUs (256x256x128 cells, 64 wells, 33.6M DOF): rank 0 builds
the global hierarchy and scatters slab plans; the 8 ranks run as threads of
this process on one GPU (a local group), and each rank's shard footprint is
the device bytes allocated by its own thread while building it (slabs, halo
plans, replicated small coarse parts, work vectors). Prints one JSON object.

    python tools/shard_footprint.py [--n 8] [--out profiles/r02/shard_footprint.json]
"""
import argparse
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2101_11649_b200 as mx  # noqa: E402

DIMS = {1: (128, 128, 64), 2: (128, 128, 128), 4: (256, 128, 128), 8: (256, 256, 128)}


def comp(n):
    d = DIMS[n]
    cells = d[0] * d[1] * d[2]
    return mx.comp_problem(*d, wells=max(1, (8 * cells) // 500000), seed=20210134)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    text = mx.load_strategy("comp_mgr_l1j")
    P1 = comp(1)
    H1 = mx.Hierarchy(mx.Matrix(P1.ptr, P1.col, P1.val), P1.partition, text, P1.unknown_map)
    one = H1.device_bytes()
    n1 = P1.n
    del H1, P1
    PN = comp(a.n)
    t0 = time.time()
    HN = mx.Hierarchy(mx.Matrix(PN.ptr, PN.col, PN.val), PN.partition, text, PN.unknown_map)
    t_setup = time.time() - t0
    glob = HN.device_bytes()
    st = mx.slab_row_starts(PN, a.n)
    g = mx.LocalGroup(a.n)
    t0 = time.time()
    with ThreadPoolExecutor(a.n) as ex:
        shards = list(ex.map(lambda r: mx.Shard(HN if r == 0 else None, r, a.n, st, group=g, scatter=True,
                                                ctx=HN.ctx), range(a.n)))
    t_scatter = time.time() - t0
    per = [s.device_bytes() for s in shards]
    rows = [s.row_end - s.row_begin for s in shards]
    out = {"config": f"cfg5 comp_mgr_l1j, N=1 {DIMS[1]} vs N={a.n} {DIMS[a.n]}",
           "n1_dofs": n1, "nN_dofs": PN.n, "rows_per_rank": rows,
           "n1_hierarchy_bytes": one, "global_hierarchy_bytes_on_rank0": glob,
           "shard_bytes_per_rank": per, "max_shard_over_n1": max(per) / one,
           "root_setup_s": t_setup, "scatter_build_s": t_scatter,
           "note": "rank 0 may drop the global hierarchy once the shards exist (the shards do not reference it); "
                   "the other ranks never hold a global operator"}
    print(json.dumps(out))
    if a.out:
        os.makedirs(os.path.dirname(a.out), exist_ok=True)
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)
    for s in shards:
        s.close()
    g.close()


if __name__ == "__main__":
    main()
