// refcpu — CPU ORACLE (test infrastructure only; see csr.hpp header).
// Restates proj/src/sparse.cpp without Eigen.
#include "csr.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace refcpu {

namespace {
int g_threads = 1;
}  // namespace

void set_threads(int n) { g_threads = n < 1 ? 1 : n; }
int threads() { return g_threads; }

Real Csr::coeff(Index i, Index j) const {
  for (Index k = ptr[i]; k < ptr[i + 1]; ++k)
    if (col[k] == j) return val[k];
  return 0.0;
}

Csr from_triplets(Index rows, Index cols, const std::vector<Triplet>& t) {
  // Stable bucket by row, then stable order by column inside a row, so equal
  // (row, col) pairs keep insertion order and are summed left to right.
  Csr A;
  A.rows = rows;
  A.cols = cols;
  std::vector<Index> cnt(static_cast<size_t>(rows) + 1, 0);
  for (const Triplet& e : t) {
    if (e.r < 0 || e.r >= rows || e.c < 0 || e.c >= cols)
      throw std::runtime_error("from_triplets: index out of range");
    ++cnt[e.r + 1];
  }
  for (Index i = 0; i < rows; ++i) cnt[i + 1] += cnt[i];
  std::vector<size_t> order(t.size());
  {
    std::vector<Index> pos(cnt.begin(), cnt.end() - 1);
    for (size_t k = 0; k < t.size(); ++k) order[pos[t[k].r]++] = k;
  }
  A.ptr.assign(static_cast<size_t>(rows) + 1, 0);
  A.col.reserve(t.size());
  A.val.reserve(t.size());
  std::vector<size_t> rowbuf;
  for (Index i = 0; i < rows; ++i) {
    rowbuf.assign(order.begin() + cnt[i], order.begin() + cnt[i + 1]);
    std::stable_sort(rowbuf.begin(), rowbuf.end(),
                     [&](size_t a, size_t b) { return t[a].c < t[b].c; });
    for (size_t q = 0; q < rowbuf.size(); ++q) {
      const Triplet& e = t[rowbuf[q]];
      if (!A.col.empty() && static_cast<Index>(A.col.size()) > A.ptr[i] && A.col.back() == e.c)
        A.val.back() = A.val.back() + e.v;
      else {
        A.col.push_back(e.c);
        A.val.push_back(e.v);
      }
    }
    A.ptr[i + 1] = static_cast<Index>(A.col.size());
  }
  return A;
}

Csr identity(Index n) {
  Csr I;
  I.rows = I.cols = n;
  I.ptr.resize(static_cast<size_t>(n) + 1);
  I.col.resize(n);
  I.val.assign(n, 1.0);
  for (Index i = 0; i <= n; ++i) I.ptr[i] = i;
  for (Index i = 0; i < n; ++i) I.col[i] = i;
  return I;
}

void validate(const Csr& A) {
  if (A.ptr.empty() || A.ptr[0] != 0) throw std::runtime_error("row_offsets[0] != 0");
  for (Index i = 0; i < A.rows; ++i) {
    if (A.ptr[i + 1] < A.ptr[i]) throw std::runtime_error("row_offsets not nondecreasing");
    Index prev = -1;
    for (Index k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
      if (A.col[k] <= prev)
        throw std::runtime_error("column indices not strictly increasing in row " + std::to_string(i));
      if (A.col[k] < 0 || A.col[k] >= A.cols)
        throw std::runtime_error("column index out of range in row " + std::to_string(i));
      if (!std::isfinite(A.val[k]))
        throw std::runtime_error("non-finite value stored in row " + std::to_string(i));
      prev = A.col[k];
    }
  }
  if (A.ptr[A.rows] != A.nnz()) throw std::runtime_error("row_offsets end != nnz");
}

// Gustavson product with Eigen's conservative accumulation: for row i, k
// ascending over A(i,:), c over B(k,:): first touch assigns B(k,c)*A(i,k),
// later touches add. Cancellation zeros are kept; columns sorted.
Csr matmul(const Csr& A, const Csr& B) {
  if (A.cols != B.rows) throw std::runtime_error("matmul: dimension mismatch");
  Csr C;
  C.rows = A.rows;
  C.cols = B.cols;
  C.ptr.assign(static_cast<size_t>(A.rows) + 1, 0);
  std::vector<std::vector<Index>> rc(A.rows);
  std::vector<std::vector<Real>> rv(A.rows);
#pragma omp parallel num_threads(g_threads)
  {
    std::vector<Index> mark(B.cols, -1);
    std::vector<Real> acc(B.cols, 0.0);
    std::vector<Index> cols;
#pragma omp for schedule(dynamic, 256)
    for (Index i = 0; i < A.rows; ++i) {
      cols.clear();
      for (Index p = A.ptr[i]; p < A.ptr[i + 1]; ++p) {
        const Index k = A.col[p];
        const Real y = A.val[p];
        for (Index q = B.ptr[k]; q < B.ptr[k + 1]; ++q) {
          const Index c = B.col[q];
          if (mark[c] != i) {
            mark[c] = i;
            acc[c] = B.val[q] * y;
            cols.push_back(c);
          } else {
            acc[c] += B.val[q] * y;
          }
        }
      }
      std::sort(cols.begin(), cols.end());
      rc[i] = cols;
      rv[i].resize(cols.size());
      for (size_t q = 0; q < cols.size(); ++q) rv[i][q] = acc[cols[q]];
    }
  }
  for (Index i = 0; i < A.rows; ++i) C.ptr[i + 1] = C.ptr[i] + static_cast<Index>(rc[i].size());
  C.col.reserve(C.ptr[A.rows]);
  C.val.reserve(C.ptr[A.rows]);
  for (Index i = 0; i < A.rows; ++i) {
    C.col.insert(C.col.end(), rc[i].begin(), rc[i].end());
    C.val.insert(C.val.end(), rv[i].begin(), rv[i].end());
  }
  return C;
}

Csr extract(const Csr& A, const IndexList& rows, const IndexList& cols) {
  std::vector<Index> cmap(A.cols, -1);
  for (size_t j = 0; j < cols.size(); ++j) {
    if (cols[j] < 0 || cols[j] >= A.cols) throw std::runtime_error("extract: column index out of range");
    cmap[cols[j]] = static_cast<Index>(j);
  }
  std::vector<Triplet> t;
  for (size_t i = 0; i < rows.size(); ++i) {
    const Index r = rows[i];
    if (r < 0 || r >= A.rows) throw std::runtime_error("extract: row index out of range");
    for (Index k = A.ptr[r]; k < A.ptr[r + 1]; ++k) {
      const Index jj = cmap[A.col[k]];
      if (jj >= 0) t.push_back({static_cast<Index>(i), jj, A.val[k]});
    }
  }
  return from_triplets(static_cast<Index>(rows.size()), static_cast<Index>(cols.size()), t);
}

IndexList complement(Index n, const IndexList& subset) {
  std::vector<char> in(n, 0);
  for (Index i : subset) in[i] = 1;
  IndexList out;
  for (Index i = 0; i < n; ++i)
    if (!in[i]) out.push_back(i);
  return out;
}

Vec diagonal(const Csr& A) {
  Vec d(A.rows, 0.0);
  for (Index i = 0; i < A.rows; ++i)
    for (Index k = A.ptr[i]; k < A.ptr[i + 1]; ++k)
      if (A.col[k] == i) d[i] = A.val[k];
  return d;
}

Vec diag_inverse(const Csr& A) {
  if (A.rows != A.cols) throw std::runtime_error("diag_inverse: matrix not square");
  Vec d(A.rows, 0.0);
  std::vector<char> present(A.rows, 0);
  for (Index i = 0; i < A.rows; ++i)
    for (Index k = A.ptr[i]; k < A.ptr[i + 1]; ++k)
      if (A.col[k] == i) {
        present[i] = 1;
        d[i] = A.val[k];
      }
  for (Index i = 0; i < A.rows; ++i) {
    if (!present[i]) throw std::runtime_error("diag_inverse: missing diagonal entry at row " + std::to_string(i));
    if (d[i] == 0.0) throw std::runtime_error("diag_inverse: zero diagonal entry at row " + std::to_string(i));
  }
  for (Index i = 0; i < A.rows; ++i) d[i] = 1.0 / d[i];
  return d;
}

bool structurally_diagonal(const Csr& A) {
  for (Index i = 0; i < A.rows; ++i)
    for (Index k = A.ptr[i]; k < A.ptr[i + 1]; ++k)
      if (A.col[k] != i) return false;
  return true;
}

void spmv_add(const Csr& A, const Vec& x, Vec& y) {
#pragma omp parallel for num_threads(g_threads) schedule(static, 4096)
  for (Index i = 0; i < A.rows; ++i) {
    Real tmp = 0.0;
    for (Index k = A.ptr[i]; k < A.ptr[i + 1]; ++k) tmp += A.val[k] * x[A.col[k]];
    y[i] += tmp;
  }
}

Vec spmv(const Csr& A, const Vec& x) {
  if (static_cast<Index>(x.size()) != A.cols) throw std::invalid_argument("spmv: dimension mismatch");
  Vec y(A.rows, 0.0);
  spmv_add(A, x, y);
  return y;
}

Csr transpose(const Csr& A) {
  Csr T;
  T.rows = A.cols;
  T.cols = A.rows;
  T.ptr.assign(static_cast<size_t>(A.cols) + 1, 0);
  for (Index k = 0; k < A.ptr[A.rows]; ++k) ++T.ptr[A.col[k] + 1];
  for (Index j = 0; j < A.cols; ++j) T.ptr[j + 1] += T.ptr[j];
  T.col.resize(A.col.size());
  T.val.resize(A.val.size());
  std::vector<Index> pos(T.ptr.begin(), T.ptr.end() - 1);
  for (Index i = 0; i < A.rows; ++i)
    for (Index k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
      const Index q = pos[A.col[k]]++;
      T.col[q] = i;
      T.val[q] = A.val[k];
    }
  return T;
}

Csr dense_to_sparse(const Dense& M) {
  std::vector<Triplet> t;
  for (Index i = 0; i < M.rows; ++i)
    for (Index j = 0; j < M.cols; ++j)
      if (M(i, j) != 0.0) t.push_back({i, j, M(i, j)});
  return from_triplets(M.rows, M.cols, t);
}

Dense to_dense(const Csr& A) {
  Dense M(A.rows, A.cols);
  for (Index i = 0; i < A.rows; ++i)
    for (Index k = A.ptr[i]; k < A.ptr[i + 1]; ++k) M(i, A.col[k]) = A.val[k];
  return M;
}

bool same_matrix(const Csr& A, const Csr& B) {
  return A.rows == B.rows && A.cols == B.cols && A.ptr == B.ptr && A.col == B.col &&
         A.val == B.val;
}

DenseLU::DenseLU(const Dense& A, Real pivot_tol) : lu_(A), n_(A.rows) {
  if (A.rows != A.cols) throw std::runtime_error("dense LU: matrix not square");
  perm_.resize(n_);
  std::iota(perm_.begin(), perm_.end(), 0);
  Dense& M = lu_;
  for (Index k = 0; k < n_; ++k) {
    Index p = k;
    Real best = std::abs(M(k, k));
    for (Index i = k + 1; i < n_; ++i)
      if (std::abs(M(i, k)) > best) {
        best = std::abs(M(i, k));
        p = i;
      }
    if (p != k) {
      for (Index j = 0; j < n_; ++j) std::swap(M(k, j), M(p, j));
      std::swap(perm_[k], perm_[p]);
    }
    const Real piv = M(k, k);
    if (piv != 0.0)
      for (Index i = k + 1; i < n_; ++i) M(i, k) /= piv;
    for (Index j = k + 1; j < n_; ++j) {
      const Real ukj = M(k, j);
      if (ukj == 0.0) continue;
      for (Index i = k + 1; i < n_; ++i) M(i, j) -= M(i, k) * ukj;
    }
  }
  for (Index i = 0; i < n_; ++i)
    if (std::abs(M(i, i)) < pivot_tol)
      throw std::runtime_error("dense LU: matrix numerically singular (pivot " + std::to_string(i) + ")");
}

Vec DenseLU::solve(const Vec& b) const {
  if (static_cast<Index>(b.size()) != n_) throw std::runtime_error("dense LU solve: dimension mismatch");
  Vec x(n_);
  for (Index i = 0; i < n_; ++i) x[i] = b[perm_[i]];
  for (Index j = 0; j < n_; ++j) {
    const Real xj = x[j];
    for (Index i = j + 1; i < n_; ++i) x[i] -= lu_(i, j) * xj;
  }
  for (Index j = n_ - 1; j >= 0; --j) {
    x[j] /= lu_(j, j);
    const Real xj = x[j];
    for (Index i = 0; i < j; ++i) x[i] -= lu_(i, j) * xj;
  }
  return x;
}

Dense DenseLU::solve(const Dense& B) const {
  Dense X(B.rows, B.cols);
  Vec col(B.rows);
  for (Index j = 0; j < B.cols; ++j) {
    for (Index i = 0; i < B.rows; ++i) col[i] = B(i, j);
    const Vec x = solve(col);
    for (Index i = 0; i < B.rows; ++i) X(i, j) = x[i];
  }
  return X;
}

DenseLU factor_dense(const Csr& A, Real pivot_tol) { return DenseLU(to_dense(A), pivot_tol); }

BlockLayout BlockLayout::from_sizes(const std::vector<Index>& sizes) {
  BlockLayout L;
  L.starts.resize(sizes.size() + 1, 0);
  for (size_t k = 0; k < sizes.size(); ++k) L.starts[k + 1] = L.starts[k] + sizes[k];
  return L;
}

BlockDiagonalLU::BlockDiagonalLU(const Csr& A, const BlockLayout& layout)
    : layout_(layout), n_(A.rows) {
  if (layout.starts.empty() || layout.starts.back() != n_)
    throw std::runtime_error("block layout does not cover the matrix");
  for (Index b = 0; b < layout.blocks(); ++b) {
    const Index lo = layout.starts[b], hi = layout.starts[b + 1];
    Dense M(hi - lo, hi - lo);
    for (Index i = lo; i < hi; ++i)
      for (Index k = A.ptr[i]; k < A.ptr[i + 1]; ++k)
        if (A.col[k] >= lo && A.col[k] < hi) M(i - lo, A.col[k] - lo) = A.val[k];
    try {
      blocks_.emplace_back(M);
    } catch (const std::exception&) {
      throw std::runtime_error("block Jacobi: singular block " + std::to_string(b));
    }
  }
}

Vec BlockDiagonalLU::solve(const Vec& r) const {
  if (static_cast<Index>(r.size()) != n_) throw std::runtime_error("block solve: dimension mismatch");
  Vec z(n_);
  for (Index b = 0; b < layout_.blocks(); ++b) {
    const Index lo = layout_.starts[b], hi = layout_.starts[b + 1];
    Vec seg(r.begin() + lo, r.begin() + hi);
    const Vec s = blocks_[b].solve(seg);
    std::copy(s.begin(), s.end(), z.begin() + lo);
  }
  return z;
}

Csr BlockDiagonalLU::solve_columns(const Csr& B) const {
  if (B.rows != n_) throw std::runtime_error("block solve: dimension mismatch");
  const Csr Bt = transpose(B);  // column access
  std::vector<Index> owner(n_);
  for (Index b = 0; b < layout_.blocks(); ++b)
    for (Index i = layout_.starts[b]; i < layout_.starts[b + 1]; ++i) owner[i] = b;
  std::vector<Triplet> out;
  for (Index c = 0; c < Bt.rows; ++c) {
    std::vector<std::pair<Index, Vec>> touched;
    for (Index k = Bt.ptr[c]; k < Bt.ptr[c + 1]; ++k) {
      const Index row = Bt.col[k];
      const Index b = owner[row];
      if (touched.empty() || touched.back().first != b)
        touched.push_back({b, Vec(layout_.starts[b + 1] - layout_.starts[b], 0.0)});
      touched.back().second[row - layout_.starts[b]] = Bt.val[k];
    }
    for (auto& [b, rhs] : touched) {
      const Vec x = blocks_[b].solve(rhs);
      for (size_t i = 0; i < x.size(); ++i)
        if (x[i] != 0.0) out.push_back({layout_.starts[b] + static_cast<Index>(i), c, x[i]});
    }
  }
  return from_triplets(n_, Bt.rows, out);
}

// Inner products use this project's canonical reduction order, which the
// device reductions of libmgrx implement too (paper_2101_11649_b200/csrc/
// krylov.cu): 592 x 256 lanes each accumulate a strided slice left to right,
// lanes fold in a fixed shuffle-down tree (offsets 16..1), warps fold in the
// same tree, and the 592 block partials fold the same way. The reference's
// order (an Eigen SIMD reduction, version unpinned) is not reproducible
// (SURVEY Appendix A.8); fixing one order makes GPU and oracle histories
// comparable bit for bit.
namespace {
constexpr int kRB = 592, kRT = 256;
Real fold32(Real* v) {
  for (int o = 16; o > 0; o >>= 1)
    for (int l = 0; l < o; ++l) v[l] = v[l] + v[l + o];
  return v[0];
}
Real fold_block(const Real* lane) {  // kRT lane values -> block value
  Real w[kRT / 32];
  Real tmp[32];
  for (int q = 0; q < kRT / 32; ++q) {
    for (int l = 0; l < 32; ++l) tmp[l] = lane[q * 32 + l];
    w[q] = fold32(tmp);
  }
  for (int l = 0; l < 32; ++l) tmp[l] = l < kRT / 32 ? w[l] : 0.0;
  return fold32(tmp);
}
}  // namespace

namespace {
int g_dot_order = 0;  // 0 canonical tree, 1 sequential, 2 Eigen SSE2 packet order
}  // namespace

void set_dot_order(int m) { g_dot_order = (m >= 0 && m <= 2) ? m : 0; }
int dot_order() { return g_dot_order; }

// Independent reduction orders (dot_order 1 and 2), used by the parity tests
// to check the north_star tolerance bar against an order the device does NOT
// share:
//  1: one accumulator, left to right (the literal loop of proj/src/krylov.cpp:
//     84-97 written as `for i: s += a_i b_i`);
//  2: the order of Eigen 3.3/3.4's vectorised redux at the x86-64 baseline the
//     reference builds for (SSE2, 2 doubles per packet; proj/CMakeLists.txt:30
//     sets no -march): two packet accumulators over alternating packets, the
//     two packets added lane-wise, one more packet if 2 remain, the two lanes
//     added, then the scalar tail left to right. Restated from knowledge of
//     Eigen's Redux.h (Eigen is not in this container), hence "unpinned".
static Real dot_sequential(const Vec& a, const Vec& b) {
  Real s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s = s + a[i] * b[i];
  return s;
}

static Real dot_eigen_sse2(const Vec& a, const Vec& b) {
  const size_t n = a.size();
  if (n < 2) return n ? a[0] * b[0] : 0.0;
  const size_t aligned = n - n % 2;  // packets of 2 doubles
  Real p0[2] = {a[0] * b[0], a[1] * b[1]};
  size_t i = 2;
  if (aligned >= 4) {
    Real p1[2] = {a[2] * b[2], a[3] * b[3]};
    const size_t end2 = aligned - aligned % 4;
    for (i = 4; i < end2; i += 4) {
      p0[0] = p0[0] + a[i] * b[i];
      p0[1] = p0[1] + a[i + 1] * b[i + 1];
      p1[0] = p1[0] + a[i + 2] * b[i + 2];
      p1[1] = p1[1] + a[i + 3] * b[i + 3];
    }
    p0[0] = p0[0] + p1[0];
    p0[1] = p0[1] + p1[1];
    if (end2 < aligned) {
      p0[0] = p0[0] + a[end2] * b[end2];
      p0[1] = p0[1] + a[end2 + 1] * b[end2 + 1];
    }
    i = aligned;
  }
  Real s = p0[0] + p0[1];
  for (; i < n; ++i) s = s + a[i] * b[i];
  return s;
}

Real dot(const Vec& a, const Vec& b) {
  if (g_dot_order == 1) return dot_sequential(a, b);
  if (g_dot_order == 2) return dot_eigen_sse2(a, b);
  const int64_t n = static_cast<int64_t>(a.size());
  const int64_t stride = static_cast<int64_t>(kRB) * kRT;
  std::vector<Real> part(kRB);
#pragma omp parallel for num_threads(g_threads) schedule(static)
  for (int blk = 0; blk < kRB; ++blk) {
    Real lane[kRT];
    for (int t = 0; t < kRT; ++t) {
      Real s = 0.0;
      for (int64_t i = static_cast<int64_t>(blk) * kRT + t; i < n; i += stride) s = s + a[i] * b[i];
      lane[t] = s;
    }
    part[blk] = fold_block(lane);
  }
  Real lane[kRT];
  for (int t = 0; t < kRT; ++t) {
    Real s = 0.0;
    for (int q = t; q < kRB; q += kRT) s = s + part[q];
    lane[t] = s;
  }
  return fold_block(lane);
}

Real norm(const Vec& a) { return std::sqrt(dot(a, a)); }

Vec sub(const Vec& a, const Vec& b) {
  Vec r(a.size());
#pragma omp parallel for num_threads(g_threads) schedule(static, 8192)
  for (int64_t i = 0; i < static_cast<int64_t>(a.size()); ++i) r[i] = a[i] - b[i];
  return r;
}

}  // namespace refcpu
