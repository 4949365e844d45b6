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
