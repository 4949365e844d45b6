"""Golden fixtures for the MGR-GMRES path.

The reference library cannot be built or imported in this environment (Eigen3,
doctest and CLI11 are absent), so the fixtures are produced by
the refcpu oracle, whose restatement is pinned by the reference's own
known-answer tests (oracle/tests/pins.cpp). They freeze, per case, a digest of
every hierarchy operator / splitting and the residual history, so any drift of
the oracle (and, in the GPU tests, of the CUDA path) is caught bit for bit.

Regenerate:  python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import refcpu  # noqa: E402
import paper_2101_11649_b200 as mx  # noqa: E402

AMG_ONLY = {"name": "amg_only", "levels": [], "coarse": {"kind": "amg_vcycle", "cycles": 1}}
AMG_ONLY_UNKNOWN = {"name": "amg_unknown", "levels": [],
                    "coarse": {"kind": "amg_vcycle", "cycles": 2, "use_unknown_map": True}}
TWO_FIELD_JACOBI = {"name": "two_field", "levels": [{"f_fields": ["f"], "interp": "jacobi",
                                                     "restrict": "injection",
                                                     "f_relax": {"kind": "jacobi", "sweeps": 2}}],
                    "coarse": {"kind": "dense_lu"}}
TWO_FIELD_RJAC = {"name": "two_field_rjac", "levels": [{"f_fields": ["f"], "interp": "jacobi",
                                                        "restrict": "jacobi",
                                                        "f_relax": {"kind": "l1_jacobi", "sweeps": 3,
                                                                    "weight": 0.8}}],
                  "coarse": {"kind": "amg_vcycle", "cycles": 2,
                             "amg": {"strength_theta": 0.25, "coarse_size": 10}}}
P_AMG_RELAX = {"name": "p_amg_relax", "levels": [{"f_fields": ["p"], "interp": "jacobi", "restrict": "injection",
                                                 "f_relax": {"kind": "amg_vcycle", "sweeps": 2,
                                                             "amg": {"coarse_size": 10}}}],
               "coarse": {"kind": "amg_vcycle", "cycles": 2, "amg": {"strength_theta": 0.1, "coarse_size": 20}}}
GLOBAL_RELAX = {"name": "global_relax", "levels": [{"f_fields": ["f"], "interp": "jacobi", "restrict": "injection",
                                                    "f_relax": {"kind": "jacobi"},
                                                    "global_relax": {"kind": "jacobi", "sweeps": 2, "weight": 0.7}}],
                "coarse": {"kind": "dense_lu"}}
# Device coverage of the non-default relaxation / transfer routes
# (proj/src/relax.cpp:55-78 hybrid partitions, :126-131 block Jacobi;
# proj/src/mgr.cpp:46-65 ideal transfers through a block layout or a dense LU).
GS_PARTITION = {"name": "gs_partition", "levels": [
    {"f_fields": ["f"], "interp": "jacobi", "restrict": "injection",
     "f_relax": {"kind": "hybrid_l1_gs_forward", "sweeps": 2,
                 "partition": [[0, 30], [30, 75], [75, 100]]},
     "global_relax": {"kind": "hybrid_l1_gs_backward", "sweeps": 1,
                      "partition": [[0, 64], [64, 130], [130, 200]]}}],
    "coarse": {"kind": "dense_lu"}}
BLOCK_IDEAL = {"name": "block_ideal", "levels": [
    {"f_fields": ["f"], "interp": "ideal", "restrict": "ideal", "ff_block_sizes": [4] * 25,
     "f_relax": {"kind": "block_jacobi_exact", "block_sizes": [5] * 20}}],
    "coarse": {"kind": "dense_lu"}}
DENSE_IDEAL = {"name": "dense_ideal", "levels": [
    {"f_fields": ["f"], "interp": "ideal", "restrict": "jacobi",
     "f_relax": {"kind": "block_jacobi_exact", "block_sizes": [10] * 10, "sweeps": 1}}],
    "coarse": {"kind": "amg_vcycle", "cycles": 1, "amg": {"coarse_size": 20}}}
DENSE_IDEAL_R = {"name": "dense_ideal_r", "levels": [
    {"f_fields": ["f"], "interp": "jacobi", "restrict": "ideal",
     "f_relax": {"kind": "l1_jacobi", "sweeps": 2}}],
    "coarse": {"kind": "dense_lu"}}


def laplace2d(nx, ny):
    rows = []
    for j in range(ny):
        for i in range(nx):
            r = {j * nx + i: 4.0}
            if i > 0: r[j * nx + i - 1] = -1.0
            if i + 1 < nx: r[j * nx + i + 1] = -1.0
            if j > 0: r[(j - 1) * nx + i] = -1.0
            if j + 1 < ny: r[(j + 1) * nx + i] = -1.0
            rows.append(r)
    return rows


def tridiag(n, lo, di, up):
    rows = []
    for i in range(n):
        r = {i: di}
        if i > 0: r[i - 1] = lo
        if i + 1 < n: r[i + 1] = up
        rows.append(r)
    return rows


def rows_to_csr(rows):
    ptr, col, val = [0], [], []
    for r in rows:
        for c in sorted(r):
            col.append(c)
            val.append(r[c])
        ptr.append(len(col))
    return np.array(ptr, np.int32), np.array(col, np.int32), np.array(val, np.float64)


def random_sdd(n, seed, extras=4):
    rng = np.random.default_rng(seed)
    rows = [dict() for _ in range(n)]
    for i in range(n):
        for _ in range(extras):
            j = int(rng.integers(0, n))
            if j != i:
                rows[i][j] = rows[i].get(j, 0.0) + float(rng.uniform(-1, 1))
    diag = 1.0 + max(sum(abs(v) for v in r.values()) for r in rows)
    for i in range(n):
        rows[i][i] = diag
    return rows


def build_problem(spec):
    """-> (ptr, col, val, fields, labels, unknown_map, rhs)"""
    kind = spec["kind"]
    if kind == "mfd":
        P = mx.mfd_problem(*spec["dims"], spec.get("field", "iid"), seed=spec.get("seed", 20210128))
        return P.ptr, P.col, P.val, P.partition.field_order, P.partition.labels, None, P.rhs
    if kind == "frac":
        P = mx.frac_problem(spec["m"], seed=spec.get("seed", 20210131))
        return P.ptr, P.col, P.val, P.partition.field_order, P.partition.labels, P.unknown_map, P.rhs
    if kind == "comp":
        P = mx.comp_problem(*spec["dims"], wells=spec.get("wells", 2), seed=spec.get("seed", 20210130))
        return P.ptr, P.col, P.val, P.partition.field_order, P.partition.labels, None, P.rhs
    rng = np.random.default_rng(spec.get("seed", 7))
    if kind == "laplace2d":
        ptr, col, val = rows_to_csr(laplace2d(*spec["dims"]))
        n = ptr.size - 1
        return ptr, col, val, ["x"], np.zeros(n, np.int32), None, rng.uniform(-1, 1, n)
    if kind == "blocksys":  # laplace2d(8,8) (+) tridiag(120,-1,2.1,-1), unknown ids 0/1
        a = laplace2d(8, 8)
        b = tridiag(120, -1.0, 2.1, -1.0)
        rows = a + [{k + len(a): v for k, v in r.items()} for r in b]
        ptr, col, val = rows_to_csr(rows)
        n = ptr.size - 1
        um = np.array([0] * len(a) + [1] * len(b), np.int32)
        return ptr, col, val, ["x"], np.zeros(n, np.int32), um, rng.uniform(-1, 1, n)
    if kind == "sdd2":  # random SDD with alternating f/c labels
        ptr, col, val = rows_to_csr(random_sdd(spec["n"], spec.get("seed", 61)))
        n = ptr.size - 1
        lab = np.array([0 if i % 2 == 0 else 1 for i in range(n)], np.int32)
        return ptr, col, val, ["f", "c"], lab, None, rng.uniform(-1, 1, n)
    raise ValueError(kind)


def strategy_text(s):
    return s if isinstance(s, str) and s.strip().startswith("{") else (
        json.dumps(s) if isinstance(s, dict) else mx.load_strategy(s))


CASES = [
    {"id": "mfd_6x5x4_mgr_pi", "problem": {"kind": "mfd", "dims": [6, 5, 4]}, "strategy": "mfd_mgr_pi",
     "rtol": 1e-8},
    {"id": "mfd_6x5x4_mgr_p", "problem": {"kind": "mfd", "dims": [6, 5, 4]}, "strategy": "mfd_mgr_p",
     "rtol": 1e-8},
    {"id": "cfg1_mgr_pi_c1", "problem": {"kind": "mfd", "dims": [20, 20, 10]}, "strategy": "mfd_mgr_pi_c1",
     "rtol": 1e-6},
    {"id": "cfg1_mgr_pi_c1_l1j", "problem": {"kind": "mfd", "dims": [20, 20, 10]},
     "strategy": "mfd_mgr_pi_c1_l1j", "rtol": 1e-6},
    {"id": "laplace_32_amg", "problem": {"kind": "laplace2d", "dims": [32, 32]}, "strategy": AMG_ONLY,
     "rtol": 1e-8},
    {"id": "blocksys_unknown_amg", "problem": {"kind": "blocksys"}, "strategy": AMG_ONLY_UNKNOWN,
     "rtol": 1e-8},
    {"id": "sdd60_two_field", "problem": {"kind": "sdd2", "n": 60}, "strategy": TWO_FIELD_JACOBI,
     "rtol": 1e-9},
    {"id": "mfd_6x5x4_p_amg_relax", "problem": {"kind": "mfd", "dims": [6, 5, 4]}, "strategy": P_AMG_RELAX,
     "rtol": 1e-8},
    {"id": "sdd200_global_relax", "problem": {"kind": "sdd2", "n": 200}, "strategy": GLOBAL_RELAX,
     "rtol": 1e-9},
    {"id": "comp_10x10x5_w2", "problem": {"kind": "comp", "dims": [10, 10, 5], "wells": 2},
     "strategy": "comp_mgr", "rtol": 1e-5},
    {"id": "comp_24x20x12_w3", "problem": {"kind": "comp", "dims": [24, 20, 12], "wells": 3},
     "strategy": "comp_mgr", "rtol": 1e-5},
    {"id": "frac_m6_mgr_u", "problem": {"kind": "frac", "m": 6}, "strategy": "frac_mgr_u", "rtol": 1e-6},
    {"id": "frac_m10_mgr_u", "problem": {"kind": "frac", "m": 10}, "strategy": "frac_mgr_u", "rtol": 1e-6},
    {"id": "sdd200_gs_partition", "problem": {"kind": "sdd2", "n": 200}, "strategy": GS_PARTITION,
     "rtol": 1e-9},
    {"id": "sdd200_block_ideal", "problem": {"kind": "sdd2", "n": 200}, "strategy": BLOCK_IDEAL,
     "rtol": 1e-9},
    {"id": "sdd200_dense_ideal", "problem": {"kind": "sdd2", "n": 200}, "strategy": DENSE_IDEAL,
     "rtol": 1e-9},
    {"id": "sdd300_dense_ideal_r", "problem": {"kind": "sdd2", "n": 300, "seed": 62}, "strategy": DENSE_IDEAL_R,
     "rtol": 1e-9},
    {"id": "sdd400_restrict_jacobi", "problem": {"kind": "sdd2", "n": 400}, "strategy": TWO_FIELD_RJAC,
     "rtol": 1e-9},
]


def digest(obj):
    h = hashlib.sha256()
    if isinstance(obj, tuple):
        for a in obj[:3]:
            h.update(np.ascontiguousarray(a).tobytes())
        h.update(repr(obj[3]).encode())
    else:
        h.update(np.ascontiguousarray(obj).tobytes())
    return h.hexdigest()[:24]


def run_case(spec, hierarchy_cls=None):
    """Build + solve with the oracle (or another implementation exposing the
    same interface); returns shape, per-path digests, iterations, history."""
    ptr, col, val, fields, labels, um, rhs = build_problem(spec["problem"])
    text = strategy_text(spec["strategy"])
    H = refcpu.RefHierarchy(ptr, col, val, fields, labels, text, um)
    info = H.info()
    digests = {p: digest(H.dump(p)) for p in refcpu.dump_paths(info)}
    _, rep = H.solve(rhs, restart=30, max_iters=500, rel_tol=spec["rtol"])
    return {"shape": info, "digests": digests, "iterations": rep["iterations"], "history": rep["history"]}


def main():
    out = {"generator": "refcpu oracle (oracle/refcpu), pinned by oracle/tests/pins.cpp", "cases": []}
    for c in CASES:
        r = run_case(c)
        out["cases"].append({"id": c["id"], "spec": c, **r})
        print(c["id"], r["shape"], r["iterations"])
    with open(os.path.join(HERE, "oracle_golden.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
