// Exact block-diagonal and dense column solves of the MGR setup and the
// block-Jacobi smoother:
//   BlockDiagonalLU (proj/src/sparse.cpp:160-223): per-block partial-pivot LU
//     of the diagonal blocks of A, solve(r), solve_columns(B);
//   ff_inverse_times dense branch (proj/src/mgr.cpp:56-61): X = A_FF^{-1} B
//     through one dense LU, then sparseView() (exact zeros dropped).
// Every block is factored and solved in the oracle's exact operation order
// (oracle/refcpu/csr_ops.cpp DenseLU: unblocked partial pivoting, first row
// of maximal |a_ik|, full-row swaps), so results are bitwise identical.
#pragma once

#include <vector>

#include "dense.cuh"

namespace mgrx {

struct BlockLU {
  int n = 0, nb = 0;
  std::vector<int> hstarts;  // host copy of the block starts (nb + 1)
  DVec<int> starts;          // block b = rows [starts[b], starts[b+1])
  DVec<long long> off;       // factors of block b at lu[off[b]], row-major s x s
  DVec<double> lu;
  DVec<int> perm;            // local row permutation of block b at perm[starts[b] ...]
  int max_size = 0;
};

// Factor the diagonal blocks of A (sizes tile [0, n)). Errors as the
// reference: "block layout does not cover the matrix", "block Jacobi:
// singular block k" (first singular block, |u_ii| < 1e-300).
void block_factor(const DCsr& A, const std::vector<int>& sizes, BlockLU& out, cudaStream_t s);
// z = blockdiag(A)^{-1} r (one thread per block).
void block_solve(const BlockLU& f, const double* r, double* z, cudaStream_t s);
// X = blockdiag(A)^{-1} B restricted to the (column, block) pairs B touches,
// exact zeros of the block solutions dropped (solve_columns).
DCsr block_solve_columns(const BlockLU& f, const DCsr& B, cudaStream_t s);
// X = A^{-1} B through the dense LU f, exact zeros dropped (sparseView).
DCsr dense_solve_columns(const DenseLU& f, const DCsr& B, cudaStream_t s);

}  // namespace mgrx
