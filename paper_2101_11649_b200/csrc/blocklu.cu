// Block-diagonal LU (block_jacobi_exact, ff_block_sizes) and the dense
// column solve of the MGR ideal transfers. See blocklu.cuh.
#include <climits>

#include "blocklu.cuh"

namespace mgrx {
namespace {

// In-place partial-pivot LU of one s x s row-major block, oracle order
// (oracle/refcpu/csr_ops.cpp DenseLU::DenseLU): pivot = first row of
// maximal |m_ik|, whole rows swapped, column scaled by the pivot (skipped
// when it is zero), trailing update skipped for zero u_kj.
__device__ void lu_inplace(int s, double* M, int* perm) {
  for (int i = 0; i < s; ++i) perm[i] = i;
  for (int k = 0; k < s; ++k) {
    int p = k;
    double best = fabs(M[k * s + k]);
    for (int i = k + 1; i < s; ++i)
      if (fabs(M[i * s + k]) > best) {
        best = fabs(M[i * s + k]);
        p = i;
      }
    if (p != k) {
      for (int j = 0; j < s; ++j) {
        const double t = M[k * s + j];
        M[k * s + j] = M[p * s + j];
        M[p * s + j] = t;
      }
      const int t = perm[k];
      perm[k] = perm[p];
      perm[p] = t;
    }
    const double piv = M[k * s + k];
    if (piv != 0.0)
      for (int i = k + 1; i < s; ++i) M[i * s + k] = __ddiv_rn(M[i * s + k], piv);
    for (int j = k + 1; j < s; ++j) {
      const double ukj = M[k * s + j];
      if (ukj == 0.0) continue;
      for (int i = k + 1; i < s; ++i) M[i * s + j] = __dsub_rn(M[i * s + j], __dmul_rn(M[i * s + k], ukj));
    }
  }
}

// x = LU^{-1} b[perm] in the oracle's order (DenseLU::solve): column-oriented
// forward elimination, then backward with the division before the updates.
__device__ void lu_solve_inplace(int s, const double* __restrict__ M, const int* __restrict__ perm,
                                 const double* __restrict__ b, double* __restrict__ x) {
  for (int i = 0; i < s; ++i) x[i] = b[perm[i]];
  for (int j = 0; j < s; ++j) {
    const double xj = x[j];
    for (int i = j + 1; i < s; ++i) x[i] = __dsub_rn(x[i], __dmul_rn(M[i * s + j], xj));
  }
  for (int j = s - 1; j >= 0; --j) {
    x[j] = __ddiv_rn(x[j], M[j * s + j]);
    const double xj = x[j];
    for (int i = 0; i < j; ++i) x[i] = __dsub_rn(x[i], __dmul_rn(M[i * s + j], xj));
  }
}

__global__ void k_block_factor(int nb, const int* __restrict__ starts, const long long* __restrict__ off,
                               const int* __restrict__ ptr, const int* __restrict__ col,
                               const double* __restrict__ val, double* __restrict__ lu, int* __restrict__ perm,
                               double tol, int* __restrict__ bad) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const int lo = starts[b], hi = starts[b + 1], s = hi - lo;
  double* M = lu + off[b];
  for (long long e = 0; e < static_cast<long long>(s) * s; ++e) M[e] = 0.0;
  for (int i = lo; i < hi; ++i)
    for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
      const int c = col[k];
      if (c >= lo && c < hi) M[(i - lo) * s + (c - lo)] = val[k];
    }
  lu_inplace(s, M, perm + lo);
  for (int i = 0; i < s; ++i)
    if (fabs(M[i * s + i]) < tol) {
      atomicMin(bad, b);
      return;
    }
}

__global__ void k_block_solve(int nb, const int* __restrict__ starts, const long long* __restrict__ off,
                              const double* __restrict__ lu, const int* __restrict__ perm,
                              const double* __restrict__ r, double* __restrict__ z) {
  pdl_enter();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const int lo = starts[b];
  lu_solve_inplace(starts[b + 1] - lo, lu + off[b], perm + lo, r + lo, z + lo);
}

// One thread per block: walk the union of the block rows' columns of B in
// ascending order (a merge over the rows' sorted column lists); for each
// column c gather the block's right-hand side (entries of B(lo:hi, c)),
// solve, and count / emit the nonzero solution entries. This is
// solve_columns (proj/src/sparse.cpp:199-223) reorganised by block: the
// same (column, block) solves with the same right-hand sides, emitted
// row-major in column order (= from_triplets of the reference's output).
template <bool kFill>
__global__ void k_block_columns(int nb, const int* __restrict__ starts, const long long* __restrict__ off,
                                const double* __restrict__ lu, const int* __restrict__ perm,
                                const int* __restrict__ bptr, const int* __restrict__ bcol,
                                const double* __restrict__ bval, int* __restrict__ head,
                                double* __restrict__ rhs, double* __restrict__ x, int* __restrict__ cnt,
                                int* __restrict__ cursor, int* __restrict__ ocol, double* __restrict__ oval) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const int lo = starts[b], hi = starts[b + 1], s = hi - lo;
  for (int i = lo; i < hi; ++i) {
    head[i] = bptr[i];
    if (!kFill) cnt[i] = 0;
  }
  while (true) {
    int c = INT_MAX;
    for (int i = lo; i < hi; ++i)
      if (head[i] < bptr[i + 1] && bcol[head[i]] < c) c = bcol[head[i]];
    if (c == INT_MAX) break;
    for (int i = lo; i < hi; ++i) {
      if (head[i] < bptr[i + 1] && bcol[head[i]] == c) {
        rhs[i] = bval[head[i]];
        ++head[i];
      } else {
        rhs[i] = 0.0;
      }
    }
    lu_solve_inplace(s, lu + off[b], perm + lo, rhs + lo, x + lo);
    for (int i = lo; i < hi; ++i) {
      if (x[i] == 0.0) continue;
      if (kFill) {
        const int o = cursor[i]++;
        ocol[o] = c;
        oval[o] = x[i];
      } else {
        ++cnt[i];
      }
    }
  }
}

__global__ void k_copy_int(int n, const int* __restrict__ a, int* __restrict__ b) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = a[i];
}

// Dense column solve: CTA c scatters row c of B^T (= column c of B) into a
// dense right-hand side and solves with the dense factors in the order of
// k_lu_solve (dense.cu) = DenseLU::solve, writing column c of X (col-major).
constexpr int kDT = 256;
__global__ void __launch_bounds__(kDT) k_dense_columns(int n, const double* __restrict__ M,
                                                       const int* __restrict__ perm,
                                                       const int* __restrict__ tptr, const int* __restrict__ tcol,
                                                       const double* __restrict__ tval, double* __restrict__ X) {
  extern __shared__ double sh[];
  double* t = sh;      // dense rhs
  double* xs = sh + n;  // solution
  const int c = blockIdx.x;
  for (int i = threadIdx.x; i < n; i += kDT) t[i] = 0.0;
  __syncthreads();
  for (int k = tptr[c] + threadIdx.x; k < tptr[c + 1]; k += kDT) t[tcol[k]] = tval[k];
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += kDT) xs[i] = t[perm[i]];
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    const double xj = xs[j];
    for (int i = j + 1 + threadIdx.x; i < n; i += kDT)
      xs[i] = __dsub_rn(xs[i], __dmul_rn(M[static_cast<size_t>(j) * n + i], xj));
    __syncthreads();
  }
  for (int j = n - 1; j >= 0; --j) {
    if (threadIdx.x == 0) xs[j] = __ddiv_rn(xs[j], M[static_cast<size_t>(j) * n + j]);
    __syncthreads();
    const double xj = xs[j];
    for (int i = threadIdx.x; i < j; i += kDT)
      xs[i] = __dsub_rn(xs[i], __dmul_rn(M[static_cast<size_t>(j) * n + i], xj));
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += kDT) X[static_cast<size_t>(c) * n + i] = xs[i];
}

// sparseView of the dense n x m col-major X, row-major CSR.
template <bool kFill>
__global__ void k_dense_sparsify(int n, int m, const double* __restrict__ X, int* __restrict__ cnt,
                                 const int* __restrict__ optr, int* __restrict__ ocol, double* __restrict__ oval) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int o = kFill ? optr[i] : 0;
  int k = 0;
  for (int c = 0; c < m; ++c) {
    const double v = X[static_cast<size_t>(c) * n + i];
    if (v == 0.0) continue;
    if (kFill) {
      ocol[o] = c;
      oval[o] = v;
      ++o;
    }
    ++k;
  }
  if (!kFill) cnt[i] = k;
}

}  // namespace

void block_factor(const DCsr& A, const std::vector<int>& sizes, BlockLU& out, cudaStream_t s) {
  const int n = A.rows;
  out.n = n;
  out.nb = static_cast<int>(sizes.size());
  out.hstarts.assign(out.nb + 1, 0);
  std::vector<long long> off(out.nb + 1, 0);
  out.max_size = 0;
  for (int b = 0; b < out.nb; ++b) {
    if (sizes[b] < 0) throw RuntimeError("block layout does not cover the matrix");
    out.hstarts[b + 1] = out.hstarts[b] + sizes[b];
    off[b + 1] = off[b] + static_cast<long long>(sizes[b]) * sizes[b];
    out.max_size = sizes[b] > out.max_size ? sizes[b] : out.max_size;
  }
  // BlockDiagonalLU ctor (proj/src/sparse.cpp:167-170)
  if (out.hstarts.back() != n) throw RuntimeError("block layout does not cover the matrix");
  out.starts.alloc(out.nb + 1, s);
  out.starts.upload(out.hstarts.data(), out.nb + 1);
  out.off.alloc(out.nb + 1, s);
  out.off.upload(off.data(), out.nb + 1);
  out.lu.alloc(off.back() > 0 ? off.back() : 1, s);
  out.perm.alloc(n > 0 ? n : 1, s);
  if (out.nb == 0) return;
  DVec<int> bad(1, s);
  const int big = INT_MAX;
  bad.upload(&big, 1);
  k_block_factor<<<blocks_for(out.nb, 128), 128, 0, s>>>(out.nb, out.starts.get(), out.off.get(), A.ptr.get(),
                                                         A.col.get(), A.val.get(), out.lu.get(), out.perm.get(),
                                                         1e-300, bad.get());
  MGRX_LAUNCH_CK();
  count_launch();
  const int b = read_scalar(bad.get(), s);
  if (b != INT_MAX) throw RuntimeError("block Jacobi: singular block " + std::to_string(b));
}

void block_solve(const BlockLU& f, const double* r, double* z, cudaStream_t s) {
  if (f.nb == 0) return;
  launch_pdl(k_block_solve, blocks_for(f.nb, 128), 128, 0, s, f.nb, f.starts.get(), f.off.get(), f.lu.get(),
             f.perm.get(), r, z);
  MGRX_LAUNCH_CK();
  count_launch();
}

DCsr block_solve_columns(const BlockLU& f, const DCsr& B, cudaStream_t s) {
  if (B.rows != f.n) throw RuntimeError("block solve: dimension mismatch");
  DCsr X;
  X.rows = B.rows;
  X.cols = B.cols;
  const int n = B.rows;
  X.ptr.alloc(n + 1, s);
  DVec<int> head(n > 0 ? n : 1, s), cnt(n > 0 ? n : 1, s), cursor(n > 0 ? n : 1, s);
  DVec<double> rhs(n > 0 ? n : 1, s), x(n > 0 ? n : 1, s);
  cnt.zero();
  const int g = blocks_for(f.nb > 0 ? f.nb : 1, 128);
  if (f.nb > 0) {
    k_block_columns<false><<<g, 128, 0, s>>>(f.nb, f.starts.get(), f.off.get(), f.lu.get(), f.perm.get(),
                                             B.ptr.get(), B.col.get(), B.val.get(), head.get(), rhs.get(),
                                             x.get(), cnt.get(), nullptr, nullptr, nullptr);
    MGRX_LAUNCH_CK();
    count_launch();
  }
  X.nnz = static_cast<int>(exclusive_scan(cnt.get(), X.ptr.get(), n, s));
  X.col.alloc(X.nnz > 0 ? X.nnz : 1, s);
  X.val.alloc(X.nnz > 0 ? X.nnz : 1, s);
  if (f.nb > 0 && n > 0) {
    k_copy_int<<<blocks_for(n, 256), 256, 0, s>>>(n, X.ptr.get(), cursor.get());
    k_block_columns<true><<<g, 128, 0, s>>>(f.nb, f.starts.get(), f.off.get(), f.lu.get(), f.perm.get(),
                                            B.ptr.get(), B.col.get(), B.val.get(), head.get(), rhs.get(),
                                            x.get(), nullptr, cursor.get(), X.col.get(), X.val.get());
    MGRX_LAUNCH_CK();
    count_launch(2);
  }
  return X;
}

DCsr dense_solve_columns(const DenseLU& f, const DCsr& B, cudaStream_t s) {
  if (B.rows != f.n) throw RuntimeError("dense LU solve: dimension mismatch");
  const int n = B.rows, m = B.cols;
  if (static_cast<double>(n) * m * 8.0 > 16e9)
    throw RuntimeError("dense ideal transfer: A_FF^{-1} B too large to form densely on the device");
  DCsr X;
  X.rows = n;
  X.cols = m;
  X.ptr.alloc(n + 1, s);
  DVec<double> Xd(static_cast<size_t>(n) * m > 0 ? static_cast<size_t>(n) * m : 1, s);
  if (n > 0 && m > 0) {
    const DCsr Bt = transpose(B, s);
    const size_t sm = 2 * sizeof(double) * n;
    if (sm > 48 * 1024)
      ensure_smem(reinterpret_cast<const void*>(k_dense_columns), static_cast<size_t>(static_cast<int>(sm)));
    k_dense_columns<<<m, kDT, sm, s>>>(n, f.lu.get(), f.perm.get(), Bt.ptr.get(), Bt.col.get(), Bt.val.get(),
                                       Xd.get());
    MGRX_LAUNCH_CK();
    count_launch();
  }
  DVec<int> cnt(n > 0 ? n : 1, s);
  if (n > 0) {
    k_dense_sparsify<false><<<blocks_for(n, 128), 128, 0, s>>>(n, m, Xd.get(), cnt.get(), nullptr, nullptr, nullptr);
    MGRX_LAUNCH_CK();
    count_launch();
  }
  X.nnz = static_cast<int>(exclusive_scan(cnt.get(), X.ptr.get(), n, s));
  X.col.alloc(X.nnz > 0 ? X.nnz : 1, s);
  X.val.alloc(X.nnz > 0 ? X.nnz : 1, s);
  if (n > 0) {
    k_dense_sparsify<true><<<blocks_for(n, 128), 128, 0, s>>>(n, m, Xd.get(), nullptr, X.ptr.get(), X.col.get(),
                                                              X.val.get());
    MGRX_LAUNCH_CK();
    count_launch();
  }
  return X;
}

}  // namespace mgrx
