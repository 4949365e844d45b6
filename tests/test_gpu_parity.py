"""GPU parity tests: the CUDA path, called through the C ABI (libmgrx.so), is
compared with the refcpu oracle on the same seeded inputs.

Bars (BASELINE.json north_star):
  * setup products (C/F splittings, P/R/A patterns and values at every level):
    bit-exact;
  * SpMV: bit-exact (per-row left-to-right order, no FMA);
  * residual history: relative gap <= 1e-10 over the first 10 entries;
  * iteration count within +-1; final true residual <= rtol.
"""
import json

import numpy as np
import pytest

import make_golden
import paper_2101_11649_b200 as mx
import refcpu

pytestmark = pytest.mark.gpu

HIST_RTOL = 1e-10


def history_close(h, hr, k=10, r0=1.0):
    """The north_star bar on residual histories (entries are ||r||/||b||):
    the first k entries agree to 1e-10 relative to the residual scale
    max(||r_k||, ||r_0||), r0 = ||b - A x0|| / ||b|| (1 for a zero guess).
    Entries reached through a large one-step reduction are ill-conditioned:
    the oracle itself, run with two inner-product orders, differs by 6.7e-9
    of the entry on golden case mfd_6x5x4_mgr_pi (1.00141048599e-05 vs
    1.00141047928e-05), so the bar cannot be "of the entry"; two
    correctly rounded fp64 runs agree to ~1e-15 of ||r_0||, which is what the
    bar checks (reduction order is unpinned)."""
    k = min(k, len(h), len(hr))
    h, hr = np.asarray(h[:k]), np.asarray(hr[:k])
    return bool(np.all(np.abs(h - hr) <= HIST_RTOL * np.maximum(np.abs(hr), r0))), (h, hr)


def _golden():
    with open(make_golden.os.path.join(make_golden.HERE, "oracle_golden.json")) as f:
        return {c["id"]: c for c in json.load(f)["cases"]}


def _same_dump(a, b):
    if isinstance(a, tuple):
        return (a[3] == b[3] and np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
                and np.array_equal(a[2].view(np.int64), b[2].view(np.int64)))
    return a.dtype == b.dtype and np.array_equal(a.view(np.int64) if a.dtype == np.float64 else a,
                                                 b.view(np.int64) if b.dtype == np.float64 else b)


@pytest.mark.parametrize("case", make_golden.CASES, ids=lambda c: c["id"])
def test_setup_bit_exact(case):
    ptr, col, val, fields, labels, um, rhs = make_golden.build_problem(case["problem"])
    text = make_golden.strategy_text(case["strategy"])
    R = refcpu.RefHierarchy(ptr, col, val, fields, labels, text, um)
    A = mx.Matrix(ptr, col, val)
    H = mx.Hierarchy(A, mx.DofPartition(fields, labels), text, um)
    assert H.info() == R.info()
    gold = _golden()[case["id"]]
    for p in refcpu.dump_paths(R.info()):
        g, r = H.dump(p), R.dump(p)
        assert _same_dump(g, r), f"{case['id']}: {p} differs from the oracle"
        assert make_golden.digest(g) == gold["digests"][p], f"{case['id']}: {p} differs from golden"


@pytest.mark.parametrize("case", make_golden.CASES, ids=lambda c: c["id"])
def test_amg_setup_info_matches_oracle(case):
    """AmgSetupInfo (level sizes, interpolation fallback rows, truncation;
    proj/include/mgrkit/amg.hpp:35-39) of every AMG in the hierarchy, through
    mgrx_amg_info, equals the oracle's."""
    ptr, col, val, fields, labels, um, rhs = make_golden.build_problem(case["problem"])
    text = make_golden.strategy_text(case["strategy"])
    R = refcpu.RefHierarchy(ptr, col, val, fields, labels, text, um)
    H = mx.Hierarchy(mx.Matrix(ptr, col, val), mx.DofPartition(fields, labels), text, um)
    info = R.info()
    which = ([-1] if info["coarse_amg_levels"] else []) + [l for l in range(info["mgr_levels"])
                                                            if info["frelax_amg_levels"][l]]
    for w in which:
        assert H.amg_info(w) == R.amg_info(w), (case["id"], w)
    with pytest.raises(mx.MgrxInvalidArgument, match="no AMG hierarchy"):
        H.amg_info(99)


@pytest.mark.parametrize("case", make_golden.CASES, ids=lambda c: c["id"])
def test_solve_parity(case):
    ptr, col, val, fields, labels, um, rhs = make_golden.build_problem(case["problem"])
    text = make_golden.strategy_text(case["strategy"])
    R = refcpu.RefHierarchy(ptr, col, val, fields, labels, text, um)
    _, rrep = R.solve(rhs, restart=30, max_iters=500, rel_tol=case["rtol"])
    A = mx.Matrix(ptr, col, val)
    H = mx.Hierarchy(A, mx.DofPartition(fields, labels), text, um)
    x, rep = H.solve(rhs, cfg=mx.KrylovConfig(restart=30, max_iters=500, rel_tol=case["rtol"], ortho="mgs"))
    assert rep.converged
    assert abs(rep.iterations - rrep["iterations"]) <= 1
    ok, detail = history_close(rep.residual_history, rrep["history"])
    assert ok, detail
    # stronger than the bar: with the canonical reduction order shared by the
    # device and the oracle, the whole GMRES run is bitwise reproducible
    assert rep.iterations == rrep["iterations"]
    assert np.array_equal(np.array(rep.residual_history), np.array(rrep["history"]))
    import scipy.sparse as sp
    M = sp.csr_matrix((val, col, ptr), shape=(ptr.size - 1,) * 2)
    assert np.linalg.norm(rhs - M @ x) <= case["rtol"] * np.linalg.norm(rhs) * (1 + 1e-9)


@pytest.mark.parametrize("case", make_golden.CASES, ids=lambda c: c["id"])
def test_solve_parity_cgs2(case):
    """The default low-synchronisation orthogonalisation (lagged CGS2,
    csrc/lowsync.cu) against the oracle in an order the device never uses
    (sequential inner products): the north_star bar — history within 1e-10
    for the first 10 steps, iterations +-1, final true residual <= rtol."""
    ptr, col, val, fields, labels, um, rhs = make_golden.build_problem(case["problem"])
    text = make_golden.strategy_text(case["strategy"])
    R = refcpu.RefHierarchy(ptr, col, val, fields, labels, text, um)
    try:
        refcpu.set_dot_order("sequential")
        _, rrep = R.solve(rhs, restart=30, max_iters=500, rel_tol=case["rtol"])
    finally:
        refcpu.set_dot_order("canonical")
    H = mx.Hierarchy(mx.Matrix(ptr, col, val), mx.DofPartition(fields, labels), text, um)
    x, rep = H.solve(rhs, cfg=mx.KrylovConfig(restart=30, max_iters=500, rel_tol=case["rtol"], ortho="cgs2"))
    assert rep.converged
    assert abs(rep.iterations - rrep["iterations"]) <= 1, (rep.iterations, rrep["iterations"])
    ok, detail = history_close(rep.residual_history, rrep["history"])
    assert ok, detail
    import scipy.sparse as sp
    M = sp.csr_matrix((val, col, ptr), shape=(ptr.size - 1,) * 2)
    assert np.linalg.norm(rhs - M @ x) <= case["rtol"] * np.linalg.norm(rhs) * (1 + 1e-9)
    # deterministic: a second solve is bitwise identical
    x2, rep2 = H.solve(rhs, cfg=mx.KrylovConfig(restart=30, max_iters=500, rel_tol=case["rtol"], ortho="cgs2"))
    assert rep2.residual_history == rep.residual_history
    assert np.array_equal(x2.view(np.int64), x.view(np.int64))


@pytest.mark.parametrize("restart,max_iters", [(1, 40), (4, 500), (7, 9), (30, 3)])
def test_cgs2_restart_and_iteration_caps(restart, max_iters):
    """Restart lengths 1..30 and max_iters hitting inside a cycle (the
    reference's loop bounds, krylov.cpp:57-60, 77): same converged flag,
    iterations +-1 and history bar as the oracle; odd n (the basis has a
    padded leading dimension)."""
    P = mx.frac_problem(8)
    assert P.n % 2 == 1, P.n
    t = mx.load_strategy("frac_mgr_u_l1j")
    R = refcpu.RefHierarchy(P.ptr, P.col, P.val, P.partition.field_order, P.partition.labels, t, P.unknown_map)
    try:
        refcpu.set_dot_order("sequential")
        _, rr = R.solve(P.rhs, restart=restart, max_iters=max_iters, rel_tol=1e-8)
    finally:
        refcpu.set_dot_order("canonical")
    H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, t, P.unknown_map)
    x, rep = H.solve(P.rhs, cfg=mx.KrylovConfig(restart=restart, max_iters=max_iters, rel_tol=1e-8, ortho="cgs2"))
    assert rep.converged == rr["converged"]
    assert abs(rep.iterations - rr["iterations"]) <= 1 and rep.iterations <= max_iters
    ok, detail = history_close(rep.residual_history, rr["history"])
    assert ok, detail
    if not rep.converged:
        assert rep.iterations == max_iters


def test_cgs2_graph_and_host_loop_agree():
    """The restart cycle as one CUDA graph (conditional WHILE node) and the
    host-driven loop (MGRX_GMRES_GRAPH=0) run the same kernels: bitwise
    equal histories and solutions."""
    import subprocess
    import sys
    code = (
        "import sys, numpy as np; sys.path.insert(0, '.');"
        "import paper_2101_11649_b200 as mx;"
        "P = mx.mfd_problem(24, 20, 12, 'layered'); t = mx.load_strategy('mfd_mgr_pi_c1_l1j');"
        "H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, t);"
        "x, rep = H.solve(P.rhs, cfg=mx.KrylovConfig(restart=30, rel_tol=1e-9, ortho='cgs2'));"
        "np.save(sys.argv[1], np.concatenate([x, rep.residual_history]));"
        "print('ok', rep.iterations, rep.gpu_launches)")
    root = make_golden.ROOT
    import tempfile
    outs = []
    for g in ("1", "0"):
        f = tempfile.mktemp(suffix=".npy")
        out = subprocess.run([sys.executable, "-c", code, f], cwd=root, capture_output=True, text=True,
                             # (two processes: the team-sum SpMV choice is a setup timing, so it
                             # is pinned off for a bitwise comparison across them)
                             env={**__import__("os").environ, "MGRX_GMRES_GRAPH": g, "MGRX_GMRES_GRAPH_DEBUG": "1",
                                  "MGRX_SPMV_VEC": "0"},
                             timeout=300)
        assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]
        assert "cycle graph disabled" not in out.stderr, out.stderr[-2000:]
        outs.append(np.load(f))
    assert np.array_equal(outs[0].view(np.int64), outs[1].view(np.int64))


def test_solve_entry_modes():
    """mgrx_solve's host / device / zero-guess paths give the same bits: x0 =
    None (MGRX_ZERO_GUESS, nothing copied for x), an explicit zero x0, a
    pinned-style `out` buffer, and device pointers; a nonzero x0 matches the
    oracle started from the same x0."""
    import torch
    P = mx.mfd_problem(12, 12, 6, "iid")
    t = mx.load_strategy("mfd_mgr_pi_c1_l1j")
    H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, t)
    cfg = mx.KrylovConfig(restart=30, rel_tol=1e-8, ortho="mgs")
    x1, r1 = H.solve(P.rhs, None, cfg)
    x2, r2 = H.solve(P.rhs, np.zeros(P.n), cfg)
    out = np.full(P.n, np.nan)
    x3, r3 = H.solve(P.rhs, None, cfg, out=out)
    assert x3 is out
    b = torch.from_numpy(P.rhs).cuda()
    xd = torch.full((P.n,), 7.0, dtype=torch.float64, device="cuda")
    xd.zero_()
    r4 = H.solve_device(b.data_ptr(), xd.data_ptr(), cfg)
    for x, r in ((x2, r2), (x3, r3), (xd.cpu().numpy(), r4)):
        assert np.array_equal(x.view(np.int64), x1.view(np.int64))
        assert r.residual_history == r1.residual_history
    x0 = np.random.default_rng(4).uniform(-1, 1, P.n)
    R = refcpu.RefHierarchy(P.ptr, P.col, P.val, P.partition.field_order, P.partition.labels, t)
    x5, r5 = H.solve(P.rhs, x0, cfg)
    xr, rr = R.solve(P.rhs, restart=30, rel_tol=1e-8, x0=x0)
    assert r5.residual_history == rr["history"]
    assert np.array_equal(x5.view(np.int64), xr.view(np.int64))
    with pytest.raises(mx.MgrxError, match="out must be"):
        H.solve(P.rhs, None, cfg, out=np.zeros(P.n, np.float32))


@pytest.mark.parametrize("case", make_golden.CASES, ids=lambda c: c["id"])
def test_apply_matches_oracle(case):
    ptr, col, val, fields, labels, um, rhs = make_golden.build_problem(case["problem"])
    text = make_golden.strategy_text(case["strategy"])
    R = refcpu.RefHierarchy(ptr, col, val, fields, labels, text, um)
    H = mx.Hierarchy(mx.Matrix(ptr, col, val), mx.DofPartition(fields, labels), text, um)
    v = np.random.default_rng(3).uniform(-1, 1, ptr.size - 1)
    z, zr = H.apply(v), R.apply(v)
    assert np.linalg.norm(z - zr) <= 1e-12 * np.linalg.norm(zr)


def test_spmv_bit_exact():
    P = mx.mfd_problem(20, 20, 10, "iid")
    A = mx.Matrix(P.ptr, P.col, P.val)
    for seed in range(3):
        x = np.random.default_rng(seed).standard_normal(P.n)
        y = A.spmv(x)
        yr = refcpu.spmv(P.ptr, P.col, P.val, x)
        assert np.array_equal(y.view(np.int64), yr.view(np.int64))
    # long rows (spanning several shared-memory chunks) and empty rows
    rng = np.random.default_rng(5)
    n = 3000
    lens = rng.integers(0, 40, n)
    lens[7] = 2900
    lens[8] = 0
    ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    col = np.concatenate([np.sort(rng.choice(n, size=l, replace=False)) for l in lens]).astype(np.int32)
    val = rng.standard_normal(ptr[-1])
    x = rng.standard_normal(n)
    y = mx.Matrix(ptr, col, val).spmv(x)
    yr = refcpu.spmv(ptr, col, val, x)
    assert np.array_equal(y.view(np.int64), yr.view(np.int64))


def test_staged_spmv_bit_exact():
    """The bulk-copy-staged SpMV (forced on, MGRX_SPMV_STAGED=2) on ragged
    large matrices: empty rows, unaligned block starts, blocks cut at the
    nonzero cap by rows of ~2000 entries, and a matrix with a row longer than
    a stage (which keeps the direct kernels)."""
    import subprocess
    import sys
    code = (
        "import sys, numpy as np; sys.path.insert(0, '.'); sys.path.insert(0, 'tests');"
        "import paper_2101_11649_b200 as mx, refcpu;"
        "rng = np.random.default_rng(11)\n"
        "for n, big in ((100003, 2000), (70001, 3000)):\n"
        "    lens = rng.integers(0, 13, n); lens[rng.integers(0, n, 40)] = 0; lens[[5, 777, n - 2]] = big\n"
        "    ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)\n"
        "    col = np.concatenate([np.sort(rng.choice(n, size=l, replace=False)) for l in lens]).astype(np.int32)\n"
        "    val = rng.standard_normal(ptr[-1]); x = rng.standard_normal(n)\n"
        "    y = mx.Matrix(ptr, col, val).spmv(x); yr = refcpu.spmv(ptr, col, val, x)\n"
        "    assert np.array_equal(y.view(np.int64), yr.view(np.int64)), n\n"
        "print('ok')")
    root = make_golden.ROOT
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                         env={**__import__("os").environ, "MGRX_SPMV_STAGED": "2"}, timeout=300)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


def test_pattern_coded_spmv_bit_exact():
    """Pattern-coded columns of the staged SpMV (forced, MGRX_SPMV_PAT=2): a
    truncated 7-point stencil with defect rows and empty rows, the hybrid-MFD
    operator (y-dependent offsets), and an irregular matrix that must fall
    back to plain column indices."""
    import subprocess
    import sys
    code = (
        "import sys, numpy as np; sys.path.insert(0, '.'); sys.path.insert(0, 'tests');"
        "import paper_2101_11649_b200 as mx, refcpu;"
        "rng = np.random.default_rng(5)\n"
        "nx, ny, nz = 37, 29, 23; n = nx * ny * nz\n"
        "rows = []\n"
        "for i in range(n):\n"
        "    x, y, z = i % nx, (i // nx) % ny, i // (nx * ny)\n"
        "    c = [i]\n"
        "    if x > 0: c.append(i - 1)\n"
        "    if x < nx - 1: c.append(i + 1)\n"
        "    if y > 0: c.append(i - nx)\n"
        "    if y < ny - 1: c.append(i + nx)\n"
        "    if z > 0: c.append(i - nx * ny)\n"
        "    if z < nz - 1: c.append(i + nx * ny)\n"
        "    if i % 997 == 0: c = []\n"
        "    if i % 1013 == 5: c = list(rng.choice(n, size=11, replace=False))\n"
        "    rows.append(np.sort(np.array(c, np.int32)))\n"
        "ptr = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int32)\n"
        "col = np.concatenate(rows).astype(np.int32)\n"
        "val = rng.standard_normal(ptr[-1]); x = rng.standard_normal(n)\n"
        "y = mx.Matrix(ptr, col, val).spmv(x); yr = refcpu.spmv(ptr, col, val, x)\n"
        "assert np.array_equal(y.view(np.int64), yr.view(np.int64)), 'stencil'\n"
        "P = mx.mfd_problem(24, 20, 12, 'layered')\n"
        "x = rng.standard_normal(P.n)\n"
        "y = mx.Matrix(P.ptr, P.col, P.val).spmv(x); yr = refcpu.spmv(P.ptr, P.col, P.val, x)\n"
        "assert np.array_equal(y.view(np.int64), yr.view(np.int64)), 'mfd'\n"
        "n = 50021; lens = rng.integers(0, 9, n)\n"
        "ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)\n"
        "col = np.concatenate([np.sort(rng.choice(n, size=l, replace=False)) for l in lens]).astype(np.int32)\n"
        "val = rng.standard_normal(ptr[-1]); x = rng.standard_normal(n)\n"
        "y = mx.Matrix(ptr, col, val).spmv(x); yr = refcpu.spmv(ptr, col, val, x)\n"
        "assert np.array_equal(y.view(np.int64), yr.view(np.int64)), 'irregular'\n"
        "print('ok')")
    root = make_golden.ROOT
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                         env={**__import__("os").environ, "MGRX_SPMV_STAGED": "2", "MGRX_SPMV_PAT": "2",
                              "MGRX_SPMV_SELL": "0", "MGRX_VERBOSE": "1"}, timeout=300)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]
    # the two structured operators took the pattern-coded plan, the irregular one did not
    assert out.stderr.count("-> staged_pat") == 2, out.stderr[-2000:]


def test_xwindow_spmv_bit_exact():
    """x-window staged SpMV (forced, MGRX_SPMV_XT=2): an irregular banded
    operator with odd column count (tail slot), empty rows and a few
    far-reaching rows; a rectangular one; and a fully random matrix whose blocks
    are cut down by the line / run caps."""
    import subprocess
    import sys
    code = (
        "import sys, numpy as np; sys.path.insert(0, '.'); sys.path.insert(0, 'tests');"
        "import paper_2101_11649_b200 as mx, refcpu;"
        "rng = np.random.default_rng(17)\n"
        "def banded(n, m):\n"
        "    rows = []\n"
        "    for i in range(n):\n"
        "        j = i * m // n\n"
        "        k = rng.integers(5, 26)\n"
        "        cand = np.concatenate([np.arange(j - 40, j + 41), np.arange(j - 5040, j - 4960), np.arange(j + 4960, j + 5040)])\n"
        "        cand = cand[(cand >= 0) & (cand < m)]\n"
        "        c = rng.choice(cand, size=min(k, len(cand)), replace=False)\n"
        "        if i % 501 == 0: c = c[:0]\n"
        "        if i % 733 == 1: c = np.concatenate([c, rng.choice(m, size=30, replace=False)])\n"
        "        if i >= n - 3: c = np.concatenate([c, [m - 1, m - 2]])\n"
        "        rows.append(np.unique(c).astype(np.int32))\n"
        "    ptr = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int32)\n"
        "    return ptr, np.concatenate(rows).astype(np.int32)\n"
        "for n, m in ((60001, 60001), (30000, 45001)):\n"
        "    ptr, col = banded(n, m)\n"
        "    val = rng.standard_normal(ptr[-1]); x = rng.standard_normal(m)\n"
        "    y = mx.Matrix(ptr, col, val, shape=(n, m)).spmv(x); yr = refcpu.spmv(ptr, col, val, x, ncols=m)\n"
        "    assert np.array_equal(y.view(np.int64), yr.view(np.int64)), (n, m)\n"
        "n = 20011; lens = rng.integers(0, 19, n)\n"
        "ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)\n"
        "col = np.concatenate([np.sort(rng.choice(n, size=l, replace=False)) for l in lens]).astype(np.int32)\n"
        "val = rng.standard_normal(ptr[-1]); x = rng.standard_normal(n)\n"
        "y = mx.Matrix(ptr, col, val).spmv(x); yr = refcpu.spmv(ptr, col, val, x)\n"
        "assert np.array_equal(y.view(np.int64), yr.view(np.int64)), 'random'\n"
        "print('ok')")
    root = make_golden.ROOT
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                         env={**__import__("os").environ, "MGRX_SPMV_XT": "2", "MGRX_VERBOSE": "1"}, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]
    assert out.stderr.count("-> xtile") == 3, out.stderr[-2000:]


def test_zero_rhs_and_errors():
    P = mx.mfd_problem(4, 4, 3, "iid")
    A = mx.Matrix(P.ptr, P.col, P.val)
    H = mx.Hierarchy(A, P.partition, mx.load_strategy("mfd_mgr_pi_c1"))
    x, rep = H.solve(np.zeros(P.n), np.ones(P.n))
    assert rep.converged and rep.iterations == 0 and not x.any()
    bad = P.rhs.copy()
    bad[3] = np.nan
    with pytest.raises(mx.MgrxError, match="non-finite"):
        H.solve(bad)
    with pytest.raises(mx.MgrxInvalidArgument, match="unknown field name: rho"):
        mx.Hierarchy(A, P.partition, json.dumps({"levels": [{"f_fields": ["rho"]}]}))
    with pytest.raises(mx.MgrxInvalidArgument, match="eliminated twice"):
        mx.Hierarchy(A, P.partition, json.dumps({"levels": [{"f_fields": ["pi"]}, {"f_fields": ["pi"]}]}))
    with pytest.raises(mx.MgrxError, match="unknown key 'bogus'"):
        mx.Hierarchy(A, P.partition, json.dumps({"coarse": {"bogus": 1}}))
    with pytest.raises(mx.MgrxInvalidArgument, match="C set is empty"):
        mx.Hierarchy(A, P.partition, json.dumps({"levels": [{"f_fields": ["p", "pi"]}]}))
    # zero diagonal in A_FF: the message names the A_FF row (proj/src/sparse.cpp:100-101)
    ptr = np.array([0, 2, 4, 5], np.int32)
    col = np.array([0, 1, 0, 1, 2], np.int32)
    val = np.array([1.0, 1.0, 1.0, 0.0, 2.0])
    with pytest.raises(mx.MgrxError, match="zero diagonal entry at row 1"):
        mx.Hierarchy(mx.Matrix(ptr, col, val), mx.DofPartition(["a", "b"], np.array([0, 0, 1], np.int32)),
                     json.dumps({"levels": [{"f_fields": ["a"]}], "coarse": {"kind": "dense_lu"}}))
    # invalid CSR is rejected like validate()
    with pytest.raises(mx.MgrxError, match="not strictly increasing in row 0"):
        mx.Matrix(np.array([0, 2, 3], np.int32), np.array([1, 0, 1], np.int32), np.ones(3))


def test_block_layout_and_partition_errors():
    """Errors of the block / dense / partitioned routes carry the reference's
    messages (proj/src/sparse.cpp:167-183, proj/src/mgr.cpp:62-64,
    proj/src/relax.cpp:12-23)."""
    ptr, col, val, fields, labels, um, rhs = make_golden.build_problem({"kind": "sdd2", "n": 200})
    A = mx.Matrix(ptr, col, val)
    part = mx.DofPartition(fields, labels)

    def lvl(**kw):
        base = {"f_fields": ["f"], "interp": "jacobi", "restrict": "injection", "f_relax": {"kind": "jacobi"}}
        base.update(kw)
        return json.dumps({"levels": [base], "coarse": {"kind": "dense_lu"}})

    with pytest.raises(mx.MgrxError, match="block layout does not cover the matrix"):
        mx.Hierarchy(A, part, lvl(interp="ideal", ff_block_sizes=[4] * 24))
    with pytest.raises(mx.MgrxError, match="block layout does not cover the matrix"):
        mx.Hierarchy(A, part, lvl(f_relax={"kind": "block_jacobi_exact", "block_sizes": [3] * 10}))
    with pytest.raises(mx.MgrxInvalidArgument, match="requires block sizes"):
        mx.Hierarchy(A, part, lvl(f_relax={"kind": "block_jacobi_exact"}))
    with pytest.raises(mx.MgrxInvalidArgument, match="partition ranges must tile"):
        mx.Hierarchy(A, part, lvl(f_relax={"kind": "hybrid_l1_gs_forward", "partition": [[0, 50], [40, 100]]}))
    with pytest.raises(mx.MgrxInvalidArgument, match="partition does not cover the matrix"):
        mx.Hierarchy(A, part, lvl(f_relax={"kind": "hybrid_l1_gs_forward", "partition": [[0, 50], [50, 99]]}))
    # a singular diagonal block (block 1 = [[1, 1], [1, 1]], nonzero diagonal)
    sp = np.array([0, 1, 2, 4, 6, 7, 8], np.int32)
    sc = np.array([0, 1, 2, 3, 2, 3, 4, 5], np.int32)
    sv = np.array([2.0, 3.0, 1.0, 1.0, 1.0, 1.0, 4.0, 5.0])
    B = mx.Matrix(sp, sc, sv)
    pb = mx.DofPartition(["f", "c"], np.array([0, 0, 0, 0, 1, 1], np.int32))
    with pytest.raises(mx.MgrxError, match="block Jacobi: singular block 1"):
        mx.Hierarchy(B, pb, json.dumps({"levels": [{"f_fields": ["f"], "f_relax": {
            "kind": "block_jacobi_exact", "block_sizes": [2, 2]}}], "coarse": {"kind": "dense_lu"}}))
    # ideal transfers with a non-diagonal A_FF, no layout and |F| > 2000
    ptr, col, val, fields, labels, um, rhs = make_golden.build_problem({"kind": "sdd2", "n": 4200})
    with pytest.raises(mx.MgrxError, match="require a structurally diagonal A_FF"):
        mx.Hierarchy(mx.Matrix(ptr, col, val), mx.DofPartition(fields, labels), lvl(interp="ideal"))


def test_identity_truncates_to_dense():
    n = 30
    ptr = np.arange(n + 1, dtype=np.int32)
    col = np.arange(n, dtype=np.int32)
    H = mx.Hierarchy(mx.Matrix(ptr, col, np.ones(n)), mx.DofPartition(["x"], np.zeros(n, np.int32)),
                     json.dumps({"coarse": {"kind": "amg_vcycle", "amg": {"coarse_size": 2}}}))
    assert H.info()["coarse_amg_levels"] == 1
    r = np.linspace(1, 30, n)
    assert np.linalg.norm(H.apply(r) - r) <= 1e-14 * np.linalg.norm(r)


@pytest.mark.parametrize("strategy", ["mfd_mgr_pi", "mfd_mgr_pi_c1", "mfd_mgr_pi_c1_l1j", "mfd_mgr_p"])
def test_cfg1_all_strategies(strategy):
    """BASELINE cfg1 (20x20x10 hybrid MFD), FGMRES(30) rtol 1e-6."""
    P = mx.mfd_problem(20, 20, 10, "iid")
    text = mx.load_strategy(strategy)
    R = refcpu.RefHierarchy(P.ptr, P.col, P.val, P.partition.field_order, P.partition.labels, text)
    _, rrep = R.solve(P.rhs, restart=30, rel_tol=1e-6)
    H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, text)
    x, rep = H.solve(P.rhs, cfg=mx.KrylovConfig(restart=30, rel_tol=1e-6))
    assert rep.converged and abs(rep.iterations - rrep["iterations"]) <= 1
    ok, detail = history_close(rep.residual_history, rrep["history"])
    assert ok, detail
    for p in refcpu.dump_paths(R.info()):
        assert _same_dump(H.dump(p), R.dump(p)), p


def test_sharded_path_device_backend_single_rank():
    """tests/slab_dist.py on the GPU backend (libmgrx slab SpMV), world size 1: the
    sharded V-cycle reproduces the library's own apply."""
    import slab_dist as D
    P = mx.mfd_problem(8, 6, 5, "iid")
    text = mx.load_strategy("mfd_mgr_pi_c1_l1j")
    H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, text)
    comm = D.Comm()
    be = D.DeviceBackend(mx.default_context())
    rr = [(0, P.n)]
    M = D.DistMgr(comm, be, H.dump, H.info(), json.loads(text), rr)
    v = np.random.default_rng(4).uniform(-1, 1, P.n)
    z = M.apply(be.vec(v)).cpu().numpy()
    zr = H.apply(v)
    assert np.linalg.norm(z - zr) <= 1e-12 * np.linalg.norm(zr)
    A = D.DistOperator(comm, be, (P.ptr, P.col, P.val), rr, rr)
    x, rep = D.gmres(comm, be, A, M.apply, be.vec(P.rhs), be.zeros(P.n), restart=30, rel_tol=1e-6)
    _, rep2 = H.solve(P.rhs, cfg=mx.KrylovConfig(restart=30, rel_tol=1e-6))
    assert rep["converged"] and abs(rep["iterations"] - rep2.iterations) <= 1


@pytest.mark.parametrize("mode", ["lv", "pipe"])
def test_alternative_gs_sweeps_are_bit_exact(mode):
    """The level-synchronous cluster sweep and the pipelined single-CTA sweep
    (MGRX_GS_MODE, read once per process) reproduce the oracle bitwise."""
    import subprocess
    import sys
    code = (
        "import sys, numpy as np; sys.path.insert(0, '.'); sys.path.insert(0, 'tests');"
        "import paper_2101_11649_b200 as mx, refcpu;"
        "P = mx.mfd_problem(20, 20, 10, 'iid'); t = mx.load_strategy('mfd_mgr_p');"
        "H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, t);"
        "R = refcpu.RefHierarchy(P.ptr, P.col, P.val, P.partition.field_order, P.partition.labels, t);"
        "v = np.random.default_rng(1).uniform(-1, 1, P.n);"
        "assert np.array_equal(H.apply(v).view(np.int64), R.apply(v).view(np.int64));"
        "x, rep = H.solve(P.rhs, cfg=mx.KrylovConfig(restart=30, rel_tol=1e-6, ortho='mgs'));"
        "_, rr = R.solve(P.rhs, restart=30, rel_tol=1e-6);"
        "assert rep.iterations == rr['iterations'] and rep.residual_history == rr['history'];"
        "print('ok')")
    root = make_golden.ROOT
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                         env={**__import__("os").environ, "MGRX_GS_MODE": mode}, timeout=300)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


@pytest.mark.parametrize("env", [{"MGRX_SPMV_BSR": "2"}, {"MGRX_SPMV_BSR": "0"}], ids=["bsr", "csr"])
def test_bsr_spmv_bit_exact(env):
    """BSR(3) storage of the 3-D elasticity displacement operators (full
    aligned 3x3 blocks, chosen per matrix by the setup timing; forced here)
    gives every row the CSR kernels' sum over the same entries in the same
    order: preconditioner application and MGS-mode history bitwise equal to
    the oracle (and to the CSR path)."""
    import subprocess
    import sys
    code = (
        "import sys, numpy as np; sys.path.insert(0, '.'); sys.path.insert(0, 'tests');"
        "import paper_2101_11649_b200 as mx, refcpu;"
        "P = mx.frac_problem(20); t = mx.load_strategy('frac_mgr_u_l1j');"
        "H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, t, P.unknown_map);"
        "R = refcpu.RefHierarchy(P.ptr, P.col, P.val, P.partition.field_order, P.partition.labels, t, P.unknown_map);"
        "v = np.random.default_rng(5).uniform(-1, 1, P.n);"
        "assert np.array_equal(H.apply(v).view(np.int64), R.apply(v).view(np.int64));"
        "x, rep = H.solve(P.rhs, cfg=mx.KrylovConfig(restart=30, rel_tol=1e-6, ortho='mgs'));"
        "xr, rr = R.solve(P.rhs, restart=30, rel_tol=1e-6);"
        "assert rep.iterations == rr['iterations'] and rep.residual_history == rr['history'];"
        "print('ok', rep.iterations)")
    root = make_golden.ROOT
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                         env={**__import__("os").environ, "MGRX_VERBOSE": "1", **env}, timeout=900)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]
    if env["MGRX_SPMV_BSR"] == "2":
        assert "bsr(3)" in out.stderr and "-> bsr" in out.stderr, out.stderr[-2000:]


@pytest.mark.parametrize("env", [{}, {"MGRX_GS_BLK_FORCE": "1"}, {"MGRX_GS_BLK_ROWS": "4096", "MGRX_GS_BLK_FORCE": "1"},
                                 {"MGRX_GS_BLK_ORDER": "local", "MGRX_GS_BLK_FORCE": "1"}, {"MGRX_GS_BLK_ROWS": "0"}],
                         ids=["autotuned", "block12288", "block4096", "blocklocal", "syncfree"])
def test_gauss_seidel_block_sweep_bit_exact(env):
    """The block-partitioned Gauss-Seidel sweep (rows cut into contiguous
    blocks, one CTA per block with its iterate in shared memory, cross-block
    dependencies polled; chosen per level at setup when it times faster) and
    the sync-free sweep (MGRX_GS_BLK_ROWS=0) reproduce the oracle bitwise: one
    preconditioner application and the whole MGS-mode residual history, on a
    system whose coarse AMG levels are large enough (196,608 / ~70K rows)."""
    import subprocess
    import sys
    code = (
        "import sys, numpy as np; sys.path.insert(0, '.'); sys.path.insert(0, 'tests');"
        "import paper_2101_11649_b200 as mx, refcpu;"
        "P = mx.mfd_problem(64, 64, 48, 'layered'); t = mx.load_strategy('mfd_mgr_pi_c1');"
        "H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, t);"
        "R = refcpu.RefHierarchy(P.ptr, P.col, P.val, P.partition.field_order, P.partition.labels, t);"
        "v = np.random.default_rng(5).uniform(-1, 1, P.n);"
        "assert np.array_equal(H.apply(v).view(np.int64), R.apply(v).view(np.int64));"
        "x, rep = H.solve(P.rhs, cfg=mx.KrylovConfig(restart=30, rel_tol=1e-6, ortho='mgs'));"
        "xr, rr = R.solve(P.rhs, restart=30, rel_tol=1e-6);"
        "assert rep.iterations == rr['iterations'] and rep.residual_history == rr['history'];"
        "assert np.array_equal(x.view(np.int64), xr.view(np.int64));"
        "print('ok', rep.iterations)")
    root = make_golden.ROOT
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                         env={**__import__("os").environ, "MGRX_VERBOSE": "1", **env}, timeout=900)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]
    if env.get("MGRX_GS_BLK_ROWS") != "0":
        assert "gs block plan" in out.stderr, out.stderr[-2000:]


@pytest.mark.parametrize("env", [{"MGRX_ARNOLDI": "0"}, {"MGRX_ARNOLDI": "1"}, {"MGRX_ARNOLDI_MERGE": "0"},
                                 {"MGRX_SPMV_STAGED": "2"}, {"MGRX_SPMV_STAGED": "0"}, {"MGRX_SPMV_SELL": "2"},
                                 {"MGRX_SPMV_SELL": "0", "MGRX_SPMV_BSR": "0"}],
                         ids=["mgs", "arnoldi", "unmerged", "staged", "direct", "sell", "nosell"])
def test_solve_paths_are_bit_exact(env):
    """Every device path choice reproduces the oracle's residual history and
    solution bitwise on a system large enough (n > 5 * 151552) that every
    Arnoldi lane owns several rows and every large operator is a staged-SpMV
    candidate: the fused persistent Arnoldi kernel vs the launch-per-
    projection MGS (MGRX_ARNOLDI), the lane-pair kernel with separate pass-1
    norm and pass-2 first-projection phases (MGRX_ARNOLDI_MERGE=0; the default
    merges them), and the bulk-copy-staged SpMV forced on
    every large matrix vs the direct kernels only (MGRX_SPMV_STAGED)."""
    import subprocess
    import sys
    code = (
        "import sys, numpy as np; sys.path.insert(0, '.'); sys.path.insert(0, 'tests');"
        "import paper_2101_11649_b200 as mx, refcpu;"
        "P = mx.mfd_problem(64, 64, 48, 'layered'); t = mx.load_strategy('mfd_mgr_pi_c1_l1j');"
        "assert P.n > 5 * 151552, P.n;"
        "H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, t);"
        "R = refcpu.RefHierarchy(P.ptr, P.col, P.val, P.partition.field_order, P.partition.labels, t);"
        "x, rep = H.solve(P.rhs, cfg=mx.KrylovConfig(restart=30, rel_tol=1e-6, ortho='mgs'));"
        "xr, rr = R.solve(P.rhs, restart=30, rel_tol=1e-6);"
        "assert rep.iterations == rr['iterations'] and rep.residual_history == rr['history'];"
        "assert np.array_equal(x.view(np.int64), xr.view(np.int64));"
        "print('ok', rep.iterations)")
    root = make_golden.ROOT
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                         env={**__import__("os").environ, **env}, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


def test_edge_cases():
    # 1x1 system, coarse dense LU only
    H = mx.Hierarchy(mx.Matrix(np.array([0, 1], np.int32), np.array([0], np.int32), np.array([4.0])),
                     mx.DofPartition(["x"], np.zeros(1, np.int32)), json.dumps({"coarse": {"kind": "dense_lu"}}))
    x, rep = H.solve(np.array([2.0]), cfg=mx.KrylovConfig(rel_tol=1e-12))
    assert rep.converged and x[0] == 0.5
    # a row without a stored diagonal in A_FF: "missing diagonal entry at row k"
    ptr = np.array([0, 1, 3, 4], np.int32)
    col = np.array([1, 0, 1, 2], np.int32)
    with pytest.raises(mx.MgrxError, match="missing diagonal entry at row 0"):
        mx.Hierarchy(mx.Matrix(ptr, col, np.ones(4)), mx.DofPartition(["a", "b"], np.array([0, 0, 1], np.int32)),
                     json.dumps({"levels": [{"f_fields": ["a"]}], "coarse": {"kind": "dense_lu"}}))
    # validation errors of the CSR boundary (proj/src/sparse.cpp:24-41)
    with pytest.raises(mx.MgrxError, match="column index out of range in row 1"):
        mx.Matrix(np.array([0, 1, 2], np.int32), np.array([0, 5], np.int32), np.ones(2))
    with pytest.raises(mx.MgrxError, match="non-finite value stored in row 0"):
        mx.Matrix(np.array([0, 1, 2], np.int32), np.array([0, 1], np.int32), np.array([np.inf, 1.0]))
    # rectangular SpMV with empty rows
    M = mx.Matrix(np.array([0, 0, 2, 2], np.int32), np.array([1, 4], np.int32), np.array([2.0, 3.0]), shape=(3, 5))
    y = M.spmv(np.arange(5, dtype=np.float64))
    assert list(y) == [0.0, 14.0, 0.0]
    # singular coarse matrix -> dense LU pivot error
    with pytest.raises(mx.MgrxError, match="numerically singular"):
        mx.Hierarchy(mx.Matrix(np.array([0, 1, 2], np.int32), np.array([0, 1], np.int32), np.array([1.0, 0.0])),
                     mx.DofPartition(["x"], np.zeros(2, np.int32)), json.dumps({"coarse": {"kind": "dense_lu"}}))


@pytest.mark.gpu
def test_amg_tail_kernel_bit_exact():
    """The single-CTA AMG tail (csrc/amgtail.cu) replaces the coarsest levels'
    launches in the l1-Jacobi strategies: one preconditioner application and
    the whole residual history stay bitwise equal to the oracle, and the tail
    is actually in use (MGRX_VERBOSE reports it)."""
    import subprocess
    import sys
    code = (
        "import sys, numpy as np; sys.path.insert(0, '.'); sys.path.insert(0, 'tests');"
        "import paper_2101_11649_b200 as mx, refcpu\n"
        "cases = [(mx.mfd_problem(20, 20, 10, 'iid'), 'mfd_mgr_pi_c1_l1j'),"
        "         (mx.comp_problem(16, 16, 8, wells=2), 'comp_mgr_l1j'), (mx.frac_problem(12), 'frac_mgr_u_l1j')]\n"
        "for P, name in cases:\n"
        "    t = mx.load_strategy(name)\n"
        "    H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, t, P.unknown_map)\n"
        "    R = refcpu.RefHierarchy(P.ptr, P.col, P.val, P.partition.field_order, P.partition.labels, t, P.unknown_map)\n"
        "    v = np.random.default_rng(3).uniform(-1, 1, P.n)\n"
        "    assert np.array_equal(H.apply(v).view(np.int64), R.apply(v).view(np.int64)), name\n"
        "    x, rep = H.solve(P.rhs, cfg=mx.KrylovConfig(restart=30, rel_tol=1e-6, ortho='mgs'))\n"
        "    _, rr = R.solve(P.rhs, restart=30, rel_tol=1e-6)\n"
        "    assert rep.iterations == rr['iterations'] and rep.residual_history == rr['history'], name\n"
        "print('ok')")
    root = make_golden.ROOT
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                         env={**__import__("os").environ, "MGRX_VERBOSE": "1"}, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]
    assert out.stderr.count("amg tail from level") >= 2, out.stderr[-3000:]
    # the cluster tail (off by default: measured slower) runs the same cases bitwise
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                         env={**__import__("os").environ, "MGRX_VERBOSE": "1", "MGRX_AMG_CTAIL": "1"}, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]
    assert out.stderr.count("amg cluster tail from level") >= 1, out.stderr[-3000:]


@pytest.mark.gpu
def test_sharded_arnoldi_mailbox_exchange_single_gpu():
    """The sharded fused Arnoldi kernel's in-kernel exchange (mailbox stores,
    system fence, per-launch tags, rank-order fold), run as a one-rank group
    that exchanges with its own mailbox (MGRX_ARNOLDI_SELFXCHG=1): every GMRES
    step goes through it and the residual history stays bitwise equal to the
    oracle's. (The multi-rank case needs one GPU per rank.)"""
    import subprocess
    import sys
    code = (
        "import sys, numpy as np; sys.path.insert(0, '.'); sys.path.insert(0, 'tests');"
        "import paper_2101_11649_b200 as mx, refcpu\n"
        "for P, name in ((mx.mfd_problem(20, 20, 10, 'iid'), 'mfd_mgr_pi_c1_l1j'),"
        "                (mx.comp_problem(16, 16, 8, wells=2), 'comp_mgr_l1j')):\n"
        "    t = mx.load_strategy(name)\n"
        "    H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, t, P.unknown_map)\n"
        "    R = refcpu.RefHierarchy(P.ptr, P.col, P.val, P.partition.field_order, P.partition.labels, t, P.unknown_map)\n"
        "    x, rep = H.solve(P.rhs, cfg=mx.KrylovConfig(restart=30, rel_tol=1e-6, ortho='mgs'))\n"
        "    _, rr = R.solve(P.rhs, restart=30, rel_tol=1e-6)\n"
        "    assert P.n % 2 == 0, P.n\n"
        "    assert rep.iterations == rr['iterations'] and rep.residual_history == rr['history'], name\n"
        "print('ok')")
    root = make_golden.ROOT
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                         env={**__import__("os").environ, "MGRX_ARNOLDI_SELFXCHG": "1"}, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]


@pytest.mark.gpu
def test_repeat_determinism_of_synchronising_kernels():
    """compute-sanitizer is closed on the GPU pool, so races are hunted by
    repetition: every kernel family with inter-CTA synchronisation (the
    low-sync sweeps' last-CTA election and conditional graph, the fused MGS
    grid barrier, the sync-free / block-partitioned / single-CTA Gauss-
    Seidel polling, the cluster dense solve, the AMG tail) reruns 25 times
    and must give the same bits every time (a race shows up as a flipped bit
    or a hang long before it shows up in a tolerance)."""
    import os
    import subprocess
    import sys
    code = (
        "import sys, numpy as np; sys.path.insert(0, '.');"
        "import paper_2101_11649_b200 as mx\n"
        "cases = [(mx.mfd_problem(32, 32, 24, 'layered'), 'mfd_mgr_pi_c1', 1e-6),"
        "         (mx.mfd_problem(24, 20, 12, 'iid'), 'mfd_mgr_pi_c1_l1j', 1e-8),"
        "         (mx.comp_problem(12, 10, 6, wells=2), 'comp_mgr', 1e-6)]\n"
        "for P, name, tol in cases:\n"
        "    H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, mx.load_strategy(name), P.unknown_map)\n"
        "    v = np.random.default_rng(1).uniform(-1, 1, P.n)\n"
        "    z0 = H.apply(v).view(np.int64)\n"
        "    ref = {}\n"
        "    for it in range(25):\n"
        "        assert np.array_equal(H.apply(v).view(np.int64), z0), (name, it)\n"
        "        for o in ('cgs2', 'mgs'):\n"
        "            x, rep = H.solve(P.rhs, cfg=mx.KrylovConfig(restart=30, rel_tol=tol, ortho=o))\n"
        "            key = (x.view(np.int64).tobytes(), tuple(rep.residual_history))\n"
        "            assert ref.setdefault(o, key) == key, (name, o, it)\n"
        "print('ok')")
    root = make_golden.ROOT
    for env in ({}, {"MGRX_GS_BLK_FORCE": "1", "MGRX_GS_BLK_ROWS": "4096"}):
        out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                             env={**os.environ, **env}, timeout=900)
        assert out.returncode == 0 and "ok" in out.stdout, (env, out.stderr[-3000:])


def _csr_matvec(ptr, col, val, x):
    y = np.zeros(ptr.size - 1)
    np.add.at(y, np.repeat(np.arange(ptr.size - 1), np.diff(ptr)), val * x[col])
    return y


@pytest.mark.parametrize("ortho", ["mgs", "cgs2"])
def test_corrupt_transfer_negative_control(ortho):
    """check_mgr_exactness (proj/src/verify.cpp:105-134) and its negative
    control (`verify --corrupt-transfer`, proj/tests/test_acceptance.cpp:25-30):
    an exact two-level MGR (ideal interpolation, dense LU on A_FF and on the
    coarse system) is a direct solver, so GMRES converges in ONE iteration to
    1e-12; with P scaled by 1.01 (mgrx_corrupt_transfer) that must fail."""
    strat = json.dumps({"levels": [{"f_fields": ["f"], "interp": "ideal", "restrict": "injection",
                                    "f_relax": {"kind": "dense_lu", "sweeps": 1}}],
                        "coarse": {"kind": "dense_lu"}})
    rng = np.random.default_rng(4711)
    cfg = mx.KrylovConfig(rel_tol=1e-12, max_iters=10, ortho=ortho)
    caught = 0
    for trial in range(12):
        n = int(rng.integers(20, 201))
        ptr, col, val = make_golden.rows_to_csr(make_golden.random_sdd(n, 1000 + trial))
        lab = (rng.uniform(size=n) < 0.5).astype(np.int32)
        lab[0], lab[1] = 0, 1  # both classes present
        part = mx.DofPartition(["f", "c"], lab)
        b = rng.uniform(-1, 1, n)
        H = mx.Hierarchy(mx.Matrix(ptr, col, val), part, strat)
        x, rep = H.solve(b, cfg=cfg)
        resid = np.linalg.norm(b - _csr_matvec(ptr, col, val, x)) / np.linalg.norm(b)
        assert rep.converged and rep.iterations == 1 and resid <= 1e-12, (trial, n, rep.iterations, resid)
        H.corrupt_transfer(0, 1.01)
        x2, rep2 = H.solve(b, cfg=cfg)
        resid2 = np.linalg.norm(b - _csr_matvec(ptr, col, val, x2)) / np.linalg.norm(b)
        if not (rep2.converged and rep2.iterations == 1 and resid2 <= 1e-12):
            caught += 1
        # the preconditioner application sees the corrupted P as well
        z_bad = H.apply(b)
        H2 = mx.Hierarchy(mx.Matrix(ptr, col, val), part, strat)
        assert not np.array_equal(z_bad, H2.apply(b))
    assert caught == 12
    with pytest.raises(mx.MgrxInvalidArgument, match="no MGR level 3"):
        H.corrupt_transfer(3, 1.01)


@pytest.mark.parametrize("code", [0, 4, 8, 16, 32, 64 + 16, 64 + 32, "tbsr"])
def test_team_sum_spmv_tolerance_mode(code):
    """Team-sum SpMV (k_spmv_vec / k_spmv_vec2: lanes share a row, fused
    multiply-adds, a shuffle tree) is the tolerance-level kernel of the
    DEFAULT solve only. Forced on for every team size and both variants
    (code 0: the setup timing's own choice, MGRX_SPMV_VEC=2) over short,
    medium and long rows:
      * mgrx_spmv without MGRX_TEAM_SUMS stays bitwise (left-to-right sums);
        with it, each row agrees with the exact sum to a few ulp of
        sum |a_ij x_j| and is deterministic run to run;
      * mgrx_apply (exact) stays bitwise equal to the oracle, the MGS-mode
        history stays identical to the oracle's, and the default-mode solve
        (every epilogue of the preconditioner through the team-sum kernels)
        meets the north_star bar (history 1e-10, iterations +-1) on the 3-D
        elasticity problem whose AMG levels have 60-200 entries per row."""
    import subprocess
    import sys
    code_txt = (
        "import sys, numpy as np; sys.path.insert(0, '.'); sys.path.insert(0, 'tests');"
        "import paper_2101_11649_b200 as mx, refcpu;"
        "rng = np.random.default_rng(11);\n"
        "for n, per in ((5000, 7), (4099, 20), (3000, 45), (2500, 130)):\n"
        "    cols = np.sort(np.stack([rng.choice(n, per, replace=False) for _ in range(n)]), axis=1).astype(np.int32)\n"
        "    ptr = (np.arange(n + 1) * per).astype(np.int32); val = rng.uniform(-1, 1, n * per)\n"
        "    A = mx.Matrix(ptr, cols.ravel(), val); x = rng.uniform(-1, 1, n)\n"
        "    prod = val.reshape(n, per) * x[cols]\n"
        "    seq = np.zeros(n)\n"
        "    for k in range(per): seq = seq + prod[:, k]\n"
        "    assert np.array_equal(A.spmv(x).view(np.int64), (0.0 + seq).view(np.int64)), (n, per)\n"
        "    yt = A.spmv(x, team_sums=True)\n"
        "    assert np.array_equal(yt.view(np.int64), A.spmv(x, team_sums=True).view(np.int64))\n"
        "    bound = 4 * np.finfo(float).eps * np.abs(prod).sum(axis=1) * np.log2(per + 1)\n"
        "    assert np.all(np.abs(yt - seq) <= bound), (n, per, np.max(np.abs(yt - seq) / bound))\n"
        "    assert not np.array_equal(yt, seq)\n"
        "nbr, nbk = 1200, 10\n"
        "bc = np.sort(np.stack([rng.choice(nbr, nbk, replace=False) for _ in range(nbr)]), axis=1)\n"
        "cols = np.repeat((3 * bc[:, None, :, None] + np.arange(3)[None, None, None, :]).reshape(nbr, 1, 3 * nbk), 3, axis=1)\n"
        "cols = cols.reshape(3 * nbr, 3 * nbk).astype(np.int32); n, per = 3 * nbr, 3 * nbk\n"
        "ptr = (np.arange(n + 1) * per).astype(np.int32); val = rng.uniform(-1, 1, n * per)\n"
        "A = mx.Matrix(ptr, cols.ravel(), val); x = rng.uniform(-1, 1, n)\n"
        "prod = val.reshape(n, per) * x[cols]\n"
        "seq = np.zeros(n)\n"
        "for k in range(per): seq = seq + prod[:, k]\n"
        "assert np.array_equal(A.spmv(x).view(np.int64), (0.0 + seq).view(np.int64))\n"
        "yt = A.spmv(x, team_sums=True)\n"
        "assert np.array_equal(yt.view(np.int64), A.spmv(x, team_sums=True).view(np.int64))\n"
        "assert np.all(np.abs(yt - seq) <= 4 * np.finfo(float).eps * np.abs(prod).sum(axis=1) * np.log2(per + 1))\n"
        "assert not np.array_equal(yt, seq)\n"
        "P = mx.frac_problem(16); t = mx.load_strategy('frac_mgr_u_l1j')\n"
        "H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, t, P.unknown_map)\n"
        "R = refcpu.RefHierarchy(P.ptr, P.col, P.val, P.partition.field_order, P.partition.labels, t, P.unknown_map)\n"
        "v = rng.uniform(-1, 1, P.n)\n"
        "assert np.array_equal(H.apply(v).view(np.int64), R.apply(v).view(np.int64))\n"
        "x, rep = H.solve(P.rhs, cfg=mx.KrylovConfig(restart=30, rel_tol=1e-6, ortho='mgs'))\n"
        "xr, rr = R.solve(P.rhs, restart=30, rel_tol=1e-6)\n"
        "assert rep.iterations == rr['iterations'] and rep.residual_history == rr['history']\n"
        "x2, rep2 = H.solve(P.rhs, cfg=mx.KrylovConfig(restart=30, rel_tol=1e-6))\n"
        "assert rep2.converged and abs(rep2.iterations - rr['iterations']) <= 1\n"
        "k = min(10, len(rep2.residual_history), len(rr['history']))\n"
        "h, hr = np.array(rep2.residual_history[:k]), np.array(rr['history'][:k])\n"
        "assert np.all(np.abs(h - hr) <= 1e-10 * np.maximum(np.abs(hr), 1.0)), (h, hr)\n"
        "print('ok', rep.iterations, rep2.iterations)\n")
    root = make_golden.ROOT
    env = {"MGRX_VERBOSE": "1", "MGRX_SPMV_VEC": "2"}
    if code == "tbsr":
        env["MGRX_SPMV_TBSR"] = "2"  # team-sum BSR(3) wherever the 3 x 3 block structure is there
    elif code:
        env["MGRX_SPMV_VEC_FORCE"] = str(code)
    out = subprocess.run([sys.executable, "-c", code_txt], cwd=root, capture_output=True, text=True,
                         env={**__import__("os").environ, **env}, timeout=900)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]
    assert "team sums (tolerance mode)" in out.stderr, out.stderr[-2000:]
    if code == "tbsr":
        assert "team-sum bsr (tolerance mode)" in out.stderr, out.stderr[-2000:]


def _newton_like_pair(seed=3):
    """Two operators of one sparsity pattern: A0 (the hierarchy is built from
    it) and A1 = A0 with every value scaled by 1 + 0.02 u, u ~ U(-1, 1)
    per entry (a later Newton step's Jacobian)."""
    P = mx.mfd_problem(8, 8, 4, "iid")
    rng = np.random.default_rng(seed)
    val1 = P.val * (1.0 + 0.02 * rng.uniform(-1.0, 1.0, P.val.size))
    return P, val1


@pytest.mark.parametrize("ortho", ["mgs", "cgs2"])
def test_solve_op_lagged_hierarchy_matches_oracle(ortho):
    """mgrx_solve_op: gmres(A1, b, x, cfg, mgr_preconditioner(H(A0))) — the
    hierarchy of an earlier Newton step kept as the preconditioner of a later
    operator (proj/include/mgrkit/krylov.hpp:33-34 takes A and M
    separately). Oracle: the same call on refcpu."""
    P, val1 = _newton_like_pair()
    text = mx.load_strategy("mfd_mgr_pi_c1")
    R = refcpu.RefHierarchy(P.ptr, P.col, P.val, P.partition.field_order, P.partition.labels, text)
    xr, rrep = R.solve_op(P.ptr, P.col, val1, P.rhs, restart=30, rel_tol=1e-8)
    ctx = mx.Context(0)
    A0, A1 = mx.Matrix(P.ptr, P.col, P.val, ctx=ctx), mx.Matrix(P.ptr, P.col, val1, ctx=ctx)
    H = mx.Hierarchy(A0, P.partition, text)
    cfg = mx.KrylovConfig(restart=30, rel_tol=1e-8, ortho=ortho)
    x, rep = mx.gmres(A1, P.rhs, None, cfg, H)
    assert rep.converged and rrep["converged"]
    assert abs(rep.iterations - rrep["iterations"]) <= 1
    ok, detail = history_close(rep.residual_history, rrep["history"])
    assert ok, detail
    if ortho == "mgs":
        assert rep.residual_history == rrep["history"]
        assert np.array_equal(x, xr)
    import scipy.sparse as sp
    M1 = sp.csr_matrix((val1, P.col, P.ptr), shape=(P.n, P.n))
    assert np.linalg.norm(P.rhs - M1 @ x) <= 1e-8 * np.linalg.norm(P.rhs) * (1 + 1e-9)
    # the lagged hierarchy is a worse preconditioner than a fresh one, not a wrong one
    _, rep0 = H.solve(P.rhs, cfg=cfg)
    assert rep0.converged and rep.iterations >= rep0.iterations
    # the hierarchy's own operator is untouched by the foreign solve, and a
    # second foreign operator (freed / re-created matrices) re-records the cycle
    del A1
    A2 = mx.Matrix(P.ptr, P.col, 0.5 * (P.val + val1), ctx=ctx)
    x2, rep2 = H.solve_op(A2, P.rhs, None, cfg)
    _, rrep2 = R.solve_op(P.ptr, P.col, 0.5 * (P.val + val1), P.rhs, restart=30, rel_tol=1e-8)
    assert rep2.converged and abs(rep2.iterations - rrep2["iterations"]) <= 1
    ok, detail = history_close(rep2.residual_history, rrep2["history"])
    assert ok, detail
    _, rep0b = H.solve(P.rhs, cfg=cfg)
    assert rep0b.residual_history == rep0.residual_history


def test_solve_op_errors():
    P, _ = _newton_like_pair()
    text = mx.load_strategy("mfd_mgr_pi_c1")
    ctx = mx.Context(0)
    H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val, ctx=ctx), P.partition, text)
    small = mx.Matrix(np.array([0, 1, 2], np.int32), np.array([0, 1], np.int32), np.ones(2), ctx=ctx)
    with pytest.raises(mx.MgrxInvalidArgument, match="mgr_apply: size mismatch"):
        H.solve_op(small, P.rhs)
    rect = mx.Matrix(np.array([0, 1, 2], np.int32), np.array([0, 2], np.int32), np.ones(2), shape=(2, 3), ctx=ctx)
    with pytest.raises(mx.MgrxInvalidArgument, match="gmres: matrix must be square"):
        H.solve_op(rect, P.rhs)
