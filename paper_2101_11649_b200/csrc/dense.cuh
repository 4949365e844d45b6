// Dense partial-pivot LU for the AMG coarsest grid and dense_lu smoothers /
// coarse solvers (proj/src/sparse.cpp:137-157). Tolerance-level parity only:
// the reference's Eigen PartialPivLU is blocked and rounds differently.
#pragma once

#include "sparse.cuh"

namespace mgrx {

struct DenseLU {
  int n = 0;
  DVec<double> lu;   // column-major n x n, unit-lower L below the diagonal, U on/above
  DVec<int> perm;    // row i of PA is row perm[i] of A
  // Block-diagonal matrices (several connected components, e.g. the MGR
  // coarse system of independent wells) are factored per component: nb > 1,
  // rows = the components' row lists back to back (each ascending), bst =
  // component starts in rows, boff = factor offsets (column-major s x s per
  // component), perm holds component-local permutations. lu is then unused.
  int nb = 1, max_block = 0;
  DVec<int> rows, bst;
  DVec<long long> boff;
  DVec<double> blu;
  // cluster solve (blocks of <= 256 rows): per-CTA slabs of 32 factor rows,
  // slab[((b * ccl + c) * slab_n + j) * 32 + r] = M_b(32c + r, j); ccl = 0: off
  int ccl = 0, slab_n = 0;
  DVec<double> slab;
  // explicit inverse of every diagonal block (blocks <= 1024 rows, <= 16M
  // entries in all): inv row-major per block at ioff[b], pblk = block of each
  // position of `rows`. Used by dense_solve(..., exact = false): a warp-per-
  // row GEMV instead of the dependent triangular sweeps. The reference's LU
  // solve is tolerance-level (Eigen's blocked order);
  // exact = true keeps the unblocked substitution (bitwise vs the oracle).
  bool has_inv = false;
  DVec<double> inv;
  DVec<long long> ioff;
  DVec<int> pblk;
};

// Densify CSR A and factor it (per connected component when A is block
// diagonal: the same operations as the dense factorization restricted to
// each block, since every cross-block entry is an exact zero); throws "dense LU: matrix numerically singular
// (pivot i)" when |u_ii| < pivot_tol.
// allow_blocks = false keeps the single dense factor (callers that read lu).
void dense_factor(const DCsr& A, DenseLU& out, cudaStream_t s, double pivot_tol = 1e-300,
                  bool allow_blocks = true);
// Build DenseLU::inv from the factors (no-op when the blocks are too large).
void dense_build_inverse(DenseLU& f, cudaStream_t s);
// x = A^{-1} b (x may alias nothing). exact = false and f.has_inv: the
// explicit-inverse GEMV (tolerance-level; see DenseLU::inv).
void dense_solve(const DenseLU& f, const double* b, double* x, cudaStream_t s, bool exact = true);

}  // namespace mgrx
