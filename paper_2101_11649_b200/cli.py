"""`python -m paper_2101_11649_b200.cli` — mirror of the reference CLI's
`generate` / `solve` / `study` subcommands (proj/tools/mgr_main.cpp:419-502)
on the B200 path.

Bundles use the reference's on-disk layout (proj/src/bundle.cpp:36-101):
matrix.mtx (Matrix Market coordinate, 17 significant digits), rhs.mtx
(array), labels.json {field_order, labels}, meta.json {problem, dofs,
unknown_map, well_rows, warnings, params}. Large bundles also get a binary
sidecar `bundle.npz` (CSR arrays, rhs, labels, unknown map) stamped with the
SHA-256 of matrix.mtx and rhs.mtx; `solve` uses it when the stamps match
(SURVEY §8f next #2), otherwise parses the Matrix Market files.

Exit codes (proj/tools/mgr_main.cpp:34): 0 converged, 1 not converged,
2 usage / invalid input, 3 internal error.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

OK, NO_CONVERGE, USAGE, INTERNAL = 0, 1, 2, 3

CONFIGS = {
    "cfg1": ("mfd", dict(nx=20, ny=20, nz=10, field="iid", seed=20210128)),
    "cfg2": ("mfd", dict(nx=128, ny=128, nz=64, field="layered", seed=20210129)),
    "cfg3": ("comp", dict(nx=100, ny=100, nz=50, wells=8, seed=20210130)),
    "cfg4": ("frac", dict(m=64, seed=20210131)),
}


class UsageError(Exception):
    pass


# ---- Matrix Market (proj/src/matrix_market.cpp) ----------------------------
def mm_write(path, ptr, col, val, ncols=None):
    n = ptr.size - 1
    rows = np.repeat(np.arange(1, n + 1), np.diff(ptr))
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix coordinate real general\n")
        f.write(f"{n} {ncols or n} {col.size}\n")
        for r, c, v in zip(rows.tolist(), (col + 1).tolist(), val.tolist()):
            f.write(f"{r} {c} {v:.17g}\n")


def mm_write_vector(path, v):
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix array real general\n")
        f.write(f"{v.size} 1\n")
        for x in v.tolist():
            f.write(f"{x:.17g}\n")


def _data_lines(f):
    for line in f:
        s = line.strip()
        if s and not s.startswith("%"):
            yield s


def mm_read(path):
    with open(path) as f:
        banner = f.readline().split()
        if len(banner) < 5 or banner[0] != "%%MatrixMarket" or banner[1].lower() != "matrix":
            raise UsageError(f"{path}:1: missing %%MatrixMarket banner")
        fmt, field, sym = banner[2].lower(), banner[3].lower(), banner[4].lower()
        if fmt != "coordinate":
            raise UsageError(f"{path}: expected coordinate format")
        if field not in ("real", "integer") or sym not in ("general", "symmetric"):
            raise UsageError(f"{path}: unsupported field/symmetry")
        lines = _data_lines(f)
        rows, cols, nnz = (int(t) for t in next(lines).split())
        data = np.loadtxt(lines, dtype=np.float64, max_rows=nnz, ndmin=2) if nnz else np.zeros((0, 3))
    i = data[:, 0].astype(np.int64) - 1
    j = data[:, 1].astype(np.int64) - 1
    v = data[:, 2].copy()
    if sym == "symmetric":
        off = i != j
        i, j, v = np.concatenate([i, j[off]]), np.concatenate([j, i[off]]), np.concatenate([v, v[off]])
    if (i < 0).any() or (i >= rows).any() or (j < 0).any() or (j >= cols).any():
        raise UsageError(f"{path}: index out of range")
    # setFromTriplets: sum duplicates in insertion order, sort columns
    order = np.lexsort((np.arange(i.size), j, i))
    i, j, v = i[order], j[order], v[order]
    key = i * cols + j
    head = np.ones(key.size, bool)
    head[1:] = key[1:] != key[:-1]
    grp = np.cumsum(head) - 1
    if head.all():
        vals = v
    else:
        vals = np.zeros(int(head.sum()))
        for k in range(v.size):  # sequential sums keep the insertion order
            vals[grp[k]] = v[k] if head[k] else vals[grp[k]] + v[k]
    ii, jj = i[head], j[head]
    ptr = np.zeros(rows + 1, np.int32)
    np.add.at(ptr, ii + 1, 1)
    return np.cumsum(ptr).astype(np.int32), jj.astype(np.int32), vals, (rows, cols)


def mm_read_vector(path):
    with open(path) as f:
        banner = f.readline().split()
        if len(banner) < 3 or banner[0] != "%%MatrixMarket":
            raise UsageError(f"{path}:1: missing %%MatrixMarket banner")
        lines = _data_lines(f)
        if banner[2].lower() == "array":
            rows, c = (int(t) for t in next(lines).split())
            if c != 1:
                raise UsageError(f"{path}: expected an n x 1 array")
            return np.array([float(next(lines)) for _ in range(rows)])
    ptr, col, val, shape = mm_read(path)
    v = np.zeros(shape[0])
    v[np.repeat(np.arange(shape[0]), np.diff(ptr))] = val
    return v


def _sha(path):
    h = hashlib.sha256()
    with open(path, "rb") as f:
        for blk in iter(lambda: f.read(1 << 24), b""):
            h.update(blk)
    return h.hexdigest()


# ---- bundles ---------------------------------------------------------------
def write_bundle(P, out, binary=True):
    os.makedirs(out, exist_ok=True)
    mm_write(os.path.join(out, "matrix.mtx"), P.ptr, P.col, P.val)
    mm_write_vector(os.path.join(out, "rhs.mtx"), P.rhs)
    with open(os.path.join(out, "labels.json"), "w") as f:
        json.dump({"field_order": P.partition.field_order, "labels": P.partition.labels.tolist()}, f)
    meta = {"problem": P.meta.get("problem", "unknown"), "dofs": int(P.n),
            "unknown_map": [] if P.unknown_map is None else P.unknown_map.tolist(),
            "well_rows": [], "warnings": [], "params": P.meta}
    with open(os.path.join(out, "meta.json"), "w") as f:
        json.dump(meta, f, indent=2)
    if binary:
        np.savez(os.path.join(out, "bundle.npz"), ptr=P.ptr, col=P.col, val=P.val, rhs=P.rhs,
                 labels=P.partition.labels,
                 umap=np.zeros(0, np.int32) if P.unknown_map is None else P.unknown_map,
                 stamp=np.frombuffer((_sha(os.path.join(out, "matrix.mtx")) +
                                      _sha(os.path.join(out, "rhs.mtx"))).encode(), np.uint8))


def read_bundle(d):
    import paper_2101_11649_b200 as mx
    for fn in ("matrix.mtx", "rhs.mtx", "labels.json", "meta.json"):
        if not os.path.exists(os.path.join(d, fn)):
            raise UsageError(f"bundle: cannot open {os.path.join(d, fn)}")
    with open(os.path.join(d, "labels.json")) as f:
        lab = json.load(f)
    with open(os.path.join(d, "meta.json")) as f:
        meta = json.load(f)
    npz = os.path.join(d, "bundle.npz")
    used_binary = False
    if os.path.exists(npz):
        z = np.load(npz)
        stamp = (_sha(os.path.join(d, "matrix.mtx")) + _sha(os.path.join(d, "rhs.mtx"))).encode()
        if bytes(z["stamp"]) == stamp:
            ptr, col, val, rhs = z["ptr"], z["col"], z["val"], z["rhs"]
            used_binary = True
    if not used_binary:
        ptr, col, val, shape = mm_read(os.path.join(d, "matrix.mtx"))
        if shape[0] != shape[1]:
            raise UsageError("bundle: matrix is not square")
        rhs = mm_read_vector(os.path.join(d, "rhs.mtx"))
    n = ptr.size - 1
    labels = np.asarray(lab["labels"], np.int32)
    fields = list(lab["field_order"])
    if rhs.size != n:
        raise UsageError("bundle: rhs length does not match matrix")
    if labels.size != n:
        raise UsageError("bundle: label count does not match matrix size")
    if labels.size and (labels.min() < 0 or labels.max() >= len(fields)):
        raise UsageError("bundle: label id out of range")
    um = meta.get("unknown_map") or None
    if um is not None:
        um = np.asarray(um, np.int32)
        if um.size != n:
            raise UsageError("bundle: unknown_map length does not match matrix size")
    return mx.Problem(ptr.astype(np.int32), col.astype(np.int32), val.astype(np.float64),
                      rhs.astype(np.float64), mx.DofPartition(fields, labels), um,
                      meta.get("params", {}) | {"problem": meta.get("problem", "unknown")})


def resolve_strategy(name, P):
    import paper_2101_11649_b200 as mx
    path = name if os.path.exists(name) else os.path.join(mx.STRATEGY_DIR, name + ".json")
    if not os.path.exists(path):
        raise UsageError(f"strategy '{name}' is neither a strategies/ name nor an existing JSON file")
    with open(path) as f:
        text = f.read()
    s = json.loads(text)
    for l, lv in enumerate(s.get("levels", [])):
        for fld in lv.get("f_fields", []):
            if fld not in P.partition.field_order:
                raise UsageError(f"strategy level {l} names field '{fld}' but the bundle has fields: "
                                 + ", ".join(P.partition.field_order))
    return text


def run_solve(P, text, sname, tol, restart, max_iters):
    import paper_2101_11649_b200 as mx
    t0 = time.perf_counter()
    H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, text, P.unknown_map)
    t1 = time.perf_counter()
    x, rep = H.solve(P.rhs, None, mx.KrylovConfig(restart=restart, max_iters=max_iters, rel_tol=tol))
    t2 = time.perf_counter()
    import scipy.sparse as sp
    A = sp.csr_matrix((P.val, P.col, P.ptr), shape=(P.n, P.n))
    bn = np.linalg.norm(P.rhs)
    true_res = float(np.linalg.norm(P.rhs - A @ x) / (bn if bn > 0 else 1.0))
    row = {"problem": P.meta.get("problem", "unknown"), "dofs": int(P.n), "strategy": sname, "tol": tol,
           "iterations": rep.iterations, "setup_seconds": t1 - t0, "solve_seconds": t2 - t1,
           "converged": bool(rep.converged), "true_residual": true_res,
           "device_setup_seconds": rep.setup_s, "device_solve_seconds": rep.solve_s,
           "dof_iters_per_s": P.n * rep.iterations / rep.solve_s if rep.solve_s > 0 else 0.0}
    return x, row


CSV_HEADER = "problem,dofs,strategy,tol,iterations,setup_seconds,solve_seconds,converged"


def csv_row(r):
    return (f"{r['problem']},{r['dofs']},{r['strategy']},{r['tol']:g},{r['iterations']},"
            f"{r['setup_seconds']:.6f},{r['solve_seconds']:.6f},{int(r['converged'])}")


def make_problem(problem, config, seed):
    import paper_2101_11649_b200 as mx
    if config in CONFIGS:
        kind, kw = CONFIGS[config]
        if kind != problem:
            raise UsageError(f"config {config} is a {kind} problem")
        kw = dict(kw)
    elif config:
        with open(config) as f:
            kw = json.load(f)
    else:
        kw = {}
    if seed is not None and seed >= 0:
        kw["seed"] = seed
    if problem == "mfd":
        return mx.mfd_problem(kw.get("nx", 8), kw.get("ny", 8), kw.get("nz", 8), kw.get("field", "iid"),
                              seed=kw.get("seed", 20210128))
    if problem == "comp":
        return mx.comp_problem(kw.get("nx", 8), kw.get("ny", 8), kw.get("nz", 8), wells=kw.get("wells", 2),
                               seed=kw.get("seed", 20210130))
    if problem == "frac":
        return mx.frac_problem(kw.get("m", 8), seed=kw.get("seed", 20210131))
    raise UsageError(f"unknown problem '{problem}' (mfd | comp | frac)")


def main(argv=None):
    ap = argparse.ArgumentParser(prog="mgrx", description="B200 MGR-GMRES: generate | solve | study")
    sub = ap.add_subparsers(dest="cmd", required=True)
    g = sub.add_parser("generate")
    g.add_argument("--problem", required=True)
    g.add_argument("--config", default="")
    g.add_argument("--seed", type=int, default=-1)
    g.add_argument("--out", required=True)
    g.add_argument("--no-binary", action="store_true")
    s = sub.add_parser("solve")
    s.add_argument("--bundle", required=True)
    s.add_argument("--strategy", required=True)
    s.add_argument("--tol", type=float, default=1e-7)
    s.add_argument("--restart", type=int, default=50)
    s.add_argument("--max-iters", type=int, default=500)
    s.add_argument("--out", default=".")
    st = sub.add_parser("study")
    st.add_argument("--problem", required=True)
    st.add_argument("--sizes", required=True)
    st.add_argument("--strategies", required=True)
    st.add_argument("--tol", type=float, default=1e-7)
    st.add_argument("--restart", type=int, default=50)
    st.add_argument("--max-iters", type=int, default=500)
    st.add_argument("--out", default=".")
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return USAGE if e.code else OK
    try:
        import paper_2101_11649_b200 as mx
        if a.cmd == "generate":
            P = make_problem(a.problem, a.config, a.seed)
            write_bundle(P, a.out, binary=not a.no_binary)
            print(f"wrote {a.problem} bundle: {P.n} dofs, fields {' '.join(P.partition.field_order)}, to {a.out}")
            return OK
        if a.cmd == "solve":
            P = read_bundle(a.bundle)
            text = resolve_strategy(a.strategy, P)
            x, row = run_solve(P, text, a.strategy, a.tol, a.restart, a.max_iters)
            os.makedirs(a.out, exist_ok=True)
            mm_write_vector(os.path.join(a.out, "x.mtx"), x)
            with open(os.path.join(a.out, "report.csv"), "w") as f:
                f.write(CSV_HEADER + "\n" + csv_row(row) + "\n")
            with open(os.path.join(a.out, "report.json"), "w") as f:
                json.dump(row, f, indent=2)
            print(CSV_HEADER + "\n" + csv_row(row))
            print(f"true residual {row['true_residual']:.3e}; solution in {a.out}/x.mtx")
            if not row["converged"]:
                print(f"solver did not converge in {row['iterations']} iterations", file=sys.stderr)
                return NO_CONVERGE
            return OK
        if a.cmd == "study":
            # proj/tools/mgr_main.cpp:344-400: sizes outer, strategies inner;
            # study.csv = report rows + "growth,<strategy>,<max/min>" lines;
            # study.json = {"rows": [...], "growth": {strategy: ratio or null}}
            sizes = []
            for tok in a.sizes.split(","):
                try:
                    sizes.append(int(tok))
                except ValueError:
                    raise UsageError(f"--sizes entry '{tok}' is not an integer")
            if len(sizes) < 2:
                raise UsageError("--sizes needs at least two refinements")
            strategies = [t for t in a.strategies.split(",") if t]
            if not strategies:
                raise UsageError("--strategies needs at least one entry")
            rows = []
            for nsz in sizes:
                P = {"mfd": lambda k: mx.mfd_problem(k, k, k, "iid"),
                     "comp": lambda k: mx.comp_problem(k, k, k, wells=2, sigma_t=1.0),  # reference default perm_sigma 1
                     "frac": lambda k: mx.frac_problem(k)}[a.problem](nsz)
                for strat in strategies:
                    _, row = run_solve(P, resolve_strategy(strat, P), strat, a.tol, a.restart, a.max_iters)
                    row["size"] = nsz
                    rows.append(row)
            csv = CSV_HEADER + "\n" + "".join(csv_row(r) + "\n" for r in rows)
            growth, all_conv = {}, True
            for strat in strategies:
                rs = [r for r in rows if r["strategy"] == strat]
                if not all(r["converged"] for r in rs):
                    csv += f"growth,{strat},unconverged\n"
                    growth[strat] = None
                    all_conv = False
                    continue
                its = [r["iterations"] for r in rs]
                growth[strat] = max(its) / max(min(its), 1)
                csv += f"growth,{strat},{growth[strat]:.4f}\n"
            os.makedirs(a.out, exist_ok=True)
            with open(os.path.join(a.out, "study.csv"), "w") as f:
                f.write(csv)
            with open(os.path.join(a.out, "study.json"), "w") as f:
                json.dump({"rows": rows, "growth": growth}, f, indent=2)
            print(csv, end="")
            return OK if all_conv else NO_CONVERGE
        return USAGE
    except UsageError as e:
        print(f"error: {e}", file=sys.stderr)
        return USAGE
    except mx.MgrxInvalidArgument as e:
        print(f"error: {e}", file=sys.stderr)
        return USAGE
    except Exception as e:  # noqa: BLE001
        print(f"internal error: {e}", file=sys.stderr)
        return INTERNAL


if __name__ == "__main__":
    sys.exit(main())
