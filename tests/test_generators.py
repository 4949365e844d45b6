"""CPU tests of the BASELINE config generators (the input side of the path)."""
import numpy as np
import scipy.sparse as sp

import paper_2101_11649_b200 as mx


def faces(nx, ny, nz):
    return (nx + 1) * ny * nz + nx * (ny + 1) * nz + nx * ny * (nz + 1)


def test_cfg1_shape_and_structure():
    P = mx.mfd_problem(20, 20, 10, "iid")
    assert P.n == 4000 + faces(20, 20, 10) == 16800
    assert P.partition.field_order == ["p", "pi"]
    assert (P.partition.labels == 0).sum() == 4000
    A = sp.csr_matrix((P.val, P.col, P.ptr), shape=(P.n, P.n))
    assert abs(A - A.T).max() == 0.0
    d = A.diagonal()
    off = np.asarray(abs(A).sum(axis=1)).ravel() - d
    assert np.all(d >= off - 1e-12 * d)  # weakly diagonally dominant (strict on cells)
    # cell rows: 7 entries; face rows: 2 (boundary) or 3 (interior)
    nnz_row = np.diff(P.ptr)
    lab = P.partition.labels
    assert np.all(nnz_row[lab == 0] == 7)
    assert set(np.unique(nnz_row[lab == 1])) == {2, 3}
    assert np.all(np.diff(P.col)[np.diff(P.ptr)[np.repeat(np.arange(P.n), np.diff(P.ptr))][1:] > 0] != 0)
    assert P.rhs.min() >= -1 and P.rhs.max() <= 1


def test_pi_block_is_diagonal_so_ideal_is_exact():
    P = mx.mfd_problem(6, 5, 4, "iid")
    A = sp.csr_matrix((P.val, P.col, P.ptr), shape=(P.n, P.n))
    f = np.where(P.partition.labels == 1)[0]
    Aff = A[f][:, f]
    assert (Aff - sp.diags(Aff.diagonal())).nnz == 0


def test_slab_major_numbering_is_contiguous():
    """Every z-layer owns one contiguous dof range, so a z-slab
    partition gives each rank a contiguous row block on every level."""
    nx, ny, nz = 5, 4, 6
    P = mx.mfd_problem(nx, ny, nz, "iid")
    slab = nx * ny + (nx + 1) * ny + nx * (ny + 1) + nx * ny
    A = sp.csr_matrix((P.val, P.col, P.ptr), shape=(P.n, P.n))
    for k in range(nz):
        lo, hi = k * slab, min((k + 1) * slab, P.n) if k < nz - 1 else P.n
        cols = A[lo:hi].indices
        # couplings reach at most the neighbouring slabs
        assert cols.min() >= max(0, lo - slab) and cols.max() < min(P.n, hi + slab)


def test_deterministic_and_seeded():
    a = mx.mfd_problem(8, 8, 4, "layered", seed=3)
    b = mx.mfd_problem(8, 8, 4, "layered", seed=3)
    c = mx.mfd_problem(8, 8, 4, "layered", seed=4)
    assert np.array_equal(a.val, b.val) and np.array_equal(a.rhs, b.rhs)
    assert not np.array_equal(a.val, c.val)


def test_layered_contrast():
    P = mx.mfd_problem(16, 16, 16, "layered", seed=20210129)
    A = sp.csr_matrix((P.val, P.col, P.ptr), shape=(P.n, P.n))
    t = -A[P.partition.labels == 0][:, P.partition.labels == 1].data
    assert t.max() / t.min() > 1e5  # per-layer ln k ~ U(-3,3) plus in-layer sigma 1.5


def test_comp_structure():
    """cfg3/cfg5 generator (BASELINE config 3): 4 unknowns
    per cell stored as cell-interleaved 4x4 blocks, a 7-point pressure
    M-matrix with ln T ~ N(0, 2^2), own-cell cross-field couplings only, rho3
    the strictly cell-local constraint, diagonally dominant density rows,
    vertical wells of nz elements x 5 dofs numbered after every cell."""
    nx, ny, nz, wells = 20, 20, 10, 3
    P = mx.comp_problem(nx, ny, nz, wells=wells)
    ncell = nx * ny * nz
    assert P.partition.field_order == ["p", "rho1", "rho2", "rho3", "well"]
    assert P.n == 4 * ncell + 5 * wells * nz
    lab = P.partition.labels
    assert np.array_equal(lab[:4 * ncell], np.tile(np.arange(4), ncell))
    assert np.all(lab[4 * ncell:] == 4)
    assert P.meta["well_elements"] == nz and P.meta["dofs_per_well_element"] == 5
    A = sp.csr_matrix((P.val, P.col, P.ptr), shape=(P.n, P.n)).tocoo()
    r, c, v = A.row, A.col, A.data
    cells = (r < 4 * ncell) & (c < 4 * ncell)
    # cross-field couplings and every rho3 entry stay inside the own cell
    cross = cells & (lab[r] != lab[c])
    assert np.all(r[cross] // 4 == c[cross] // 4)
    rho3 = cells & (lab[r] == 3)
    assert np.all(r[rho3] // 4 == c[rho3] // 4)
    # 7-point pressure M-matrix: p-p off-diagonals negative, at most 6 per row
    pp = cells & (lab[r] == 0) & (lab[c] == 0) & (r != c)
    assert np.all(v[pp] < 0)
    assert np.bincount(r[pp] // 4, minlength=ncell).max() == 6
    lnT = np.log(-v[pp])
    assert 1.8 < lnT.std() < 2.2 and abs(lnT.mean()) < 0.2
    d = A.tocsr().diagonal()
    offpp = np.bincount(r[pp], weights=-v[pp], minlength=P.n)
    prow = np.arange(0, 4 * ncell, 4)
    assert np.all(d[prow] >= offpp[prow])
    # density blocks (same-field entries of the rho1/rho2 rows) strictly diagonally dominant
    dens = cells & ((lab[r] == 1) | (lab[r] == 2)) & (lab[c] == lab[r]) & (r != c)
    off = np.bincount(r[dens], weights=np.abs(v[dens]), minlength=P.n)
    drow = np.where((lab == 1) | (lab == 2))[0]
    assert np.all(np.abs(d[drow]) > off[drow])
    # wells couple to well dofs and to their perforated cells' p, rho1, rho2
    # (never to the rho3 constraint); one perforated cell per element below
    # the control element (e = 0, the rate-control row with a stored zero
    # diagonal, like the reference's control rows)
    wr = r >= 4 * ncell
    assert np.all((c[wr] >= 4 * ncell) | (lab[c[wr]] <= 2))
    perf = np.unique(c[wr & (c < 4 * ncell)] // 4)
    assert perf.size == wells * (nz - 1)


def test_frac_structure():
    """cfg4 generator (BASELINE config 4): 3-D Q1 elasticity on
    m^3 nodes with the bottom and top node planes fixed, a mid-plane
    fracture of (m-1)^2 pressure elements whose interior plane nodes are
    duplicated; node-interleaved displacement dofs with the component as the
    unknown map; 81 entries on interior displacement rows; symmetric A_uu."""
    m = 8
    P = mx.frac_problem(m)
    assert P.partition.field_order == ["u", "p"]
    nodes = m * m * (m - 2) + (m - 2) ** 2
    nfrac = (m - 1) ** 2
    assert P.n == 3 * nodes + nfrac
    lab = P.partition.labels
    assert np.all(lab[:3 * nodes] == 0) and np.all(lab[3 * nodes:] == 1)
    assert np.array_equal(P.unknown_map[:3 * nodes], np.tile(np.arange(3), nodes))
    assert np.all(P.unknown_map[3 * nodes:] == 0)
    A = sp.csr_matrix((P.val, P.col, P.ptr), shape=(P.n, P.n))
    u = np.arange(3 * nodes)
    Auu = A[u][:, u]
    assert abs(Auu - Auu.T).max() == 0.0
    assert np.all(A.diagonal() > 0)
    per_row = np.diff(P.ptr)[:3 * nodes]
    assert per_row.max() == 81 and (per_row == 81).sum() >= 3 * (m - 4) ** 3  # interior: 27 neighbours x 3
    # full-size point: 64^3 nodes -> 777,357 dofs
    assert 3 * (64 * 64 * 62 + 62 * 62) + 63 * 63 == 777357
