// refcpu — CPU ORACLE for the MGR-GMRES hot path. TEST INFRASTRUCTURE ONLY.
//
// This is an Eigen-free restatement of the reference mgrkit library
// (/root/reference/proj/src/*.cpp, which cannot be compiled here: Eigen3,
// doctest and CLI11 are absent). Only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py may load it. The product
// (libmgrx) never links or calls anything under oracle/.
//
// Numerics contract: fp64, int32 indices, no FMA
// (built with -ffp-contract=off), per-row left-to-right SpMV, Eigen
// "conservative" SpGEMM accumulation order, setFromTriplets duplicate order.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace refcpu {

using Real = double;
using Index = int;
using Vec = std::vector<Real>;
using IndexList = std::vector<Index>;

struct Triplet {
  Index r, c;
  Real v;
};

// Compressed sparse row matrix; columns strictly increasing per row.
// Mirrors the Eigen RowMajor SparseMatrix used by the reference
// (proj/include/mgrkit/types.hpp:20).
struct Csr {
  Index rows = 0, cols = 0;
  std::vector<Index> ptr{0};
  std::vector<Index> col;
  std::vector<Real> val;
  int64_t nnz() const { return static_cast<int64_t>(col.size()); }
  Real coeff(Index i, Index j) const;
};

// Dense column-major matrix helper.
struct Dense {
  Index rows = 0, cols = 0;
  std::vector<Real> a;  // column major
  Dense() = default;
  Dense(Index r, Index c) : rows(r), cols(c), a(static_cast<size_t>(r) * c, 0.0) {}
  Real& operator()(Index i, Index j) { return a[static_cast<size_t>(j) * rows + i]; }
  Real operator()(Index i, Index j) const { return a[static_cast<size_t>(j) * rows + i]; }
};

// setFromTriplets semantics (proj/src/sparse.cpp:10-15): duplicates summed in
// insertion order, explicit zeros kept, columns sorted.
Csr from_triplets(Index rows, Index cols, const std::vector<Triplet>& t);
Csr identity(Index n);
void validate(const Csr& A);                                   // sparse.cpp:24-41
Csr matmul(const Csr& A, const Csr& B);                        // sparse.cpp:43-49
Csr extract(const Csr& A, const IndexList& rows, const IndexList& cols);  // 51-67
IndexList complement(Index n, const IndexList& subset);        // 69-77
Vec diagonal(const Csr& A);                                    // 79-85
Vec diag_inverse(const Csr& A);                                // 87-104
bool structurally_diagonal(const Csr& A);                      // 118-123
Vec spmv(const Csr& A, const Vec& x);                          // 126-129
// y <- y + A x  (Eigen "y += A*x", row sums left to right then added)
void spmv_add(const Csr& A, const Vec& x, Vec& y);
Csr transpose(const Csr& A);                                   // 131-135
Csr dense_to_sparse(const Dense& M);                           // sparseView(): drops exact 0
Dense to_dense(const Csr& A);
bool same_matrix(const Csr& A, const Csr& B);

// Partial-pivot dense LU (proj/src/sparse.cpp:137-157). Tolerance-level
// parity only: Eigen's blocked PartialPivLU rounds differently.
class DenseLU {
 public:
  DenseLU() = default;
  explicit DenseLU(const Dense& A, Real pivot_tol = 1e-300);
  Vec solve(const Vec& b) const;
  Dense solve(const Dense& B) const;
  Index size() const { return n_; }

 private:
  Dense lu_;
  std::vector<Index> perm_;  // row i of PA = row perm_[i] of A
  Index n_ = 0;
};
DenseLU factor_dense(const Csr& A, Real pivot_tol = 1e-300);

struct BlockLayout {
  std::vector<Index> starts;
  Index blocks() const { return static_cast<Index>(starts.size()) - 1; }
  static BlockLayout from_sizes(const std::vector<Index>& sizes);
};

// proj/src/sparse.cpp:167-223
class BlockDiagonalLU {
 public:
  BlockDiagonalLU() = default;
  BlockDiagonalLU(const Csr& A, const BlockLayout& layout);
  Vec solve(const Vec& r) const;
  Csr solve_columns(const Csr& B) const;

 private:
  std::vector<DenseLU> blocks_;
  BlockLayout layout_;
  Index n_ = 0;
};

// Vector helpers (Eigen expression semantics, elementwise, no FMA).
Real dot(const Vec& a, const Vec& b);
Real norm(const Vec& a);
Vec sub(const Vec& a, const Vec& b);

// Number of OpenMP threads used by the row-parallel kernels (1 = faithful
// serial reference). Results never depend on it.
void set_threads(int n);
// inner-product order of dot()/norm(): 0 canonical (device) tree, 1 sequential,
// 2 Eigen SSE2 packet order (see csr_ops.cpp)
void set_dot_order(int m);
int dot_order();
int threads();

}  // namespace refcpu
