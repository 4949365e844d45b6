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
};

// Densify CSR A and factor it; throws "dense LU: matrix numerically singular
// (pivot i)" when |u_ii| < pivot_tol.
void dense_factor(const DCsr& A, DenseLU& out, cudaStream_t s, double pivot_tol = 1e-300);
// x = A^{-1} b (x may alias nothing).
void dense_solve(const DenseLU& f, const double* b, double* x, cudaStream_t s);

}  // namespace mgrx
