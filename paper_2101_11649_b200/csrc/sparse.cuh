// Device-resident CSR (fp64 values, int32 indices) and the sparse kernels of
// the MGR-GMRES path. Setup kernels are bit-exact restatements of the
// reference's Eigen semantics; every floating-point
// operation is an explicit __dmul_rn/__dadd_rn/__dsub_rn/__ddiv_rn and the
// library is compiled with --fmad=false, so no contraction can change a bit.
#pragma once

#include "common.cuh"

namespace mgrx {

struct DCsr {
  int rows = 0, cols = 0, nnz = 0;
  DVec<int> ptr, col;
  DVec<double> val;
  // Staged-SpMV block plan (spmv_prepare): nblk row blocks, plan holds the
  // nblk+1 first rows then the nblk+1 first nonzeros. nblk == 0: no plan.
  int nblk = 0;
  DVec<int> plan;
  // plan kind: 0 staged (<= 256 rows / 2048 entries per block), 1 warp-
  // specialised long-row kernel (<= 64 rows / 2048 entries per block)
  int plan_kind = 0;
  // warp-specialised plan kept alongside for the Jacobi-sweep epilogues
  // (their two gathers per entry make the product pass the long pole, which
  // the specialised kernel overlaps with the sums): nblk_w == 0: none
  int nblk_w = 0;
  DVec<int> plan_w;
  // BSR copy (spmv_prepare, when every block row of b rows holds full,
  // aligned b x b blocks with identical column patterns, and it times
  // faster): bptr per block row, bcol per block (block column), bval b*b
  // values per block, row-major inside the block -- the same entries in the
  // same per-row order as the CSR, so row sums are bitwise equal. bplan:
  // first block row of each CTA chunk (nbchunk + 1). bsr == 0: none.
  int bsr = 0, nbchunk = 0;
  DVec<int> bptr, bcol, bplan;
  DVec<double> bval;
  // SELL-32 copy (medium rows; chosen per matrix by the setup timing): rows
  // length-sorted inside windows of 256, slices of 32 rows stored column-
  // major (slot k of lane l at soff[slice] + 32 k + l), each row's entries in
  // its CSR order; sperm = original row of a slot, slen = its length.
  // nslice == 0: none.
  int nslice = 0;
  DVec<int> soff, sperm, slen, scol;
  DVec<double> sval;
  // Pattern-coded columns of the staged plan (spmv_prepare; stencil-like
  // operators): inside a row block, rows whose column offsets col - row agree
  // share one dictionary entry. Per block: pmeta = {first dictionary int
  // (multiple of 4), dictionary row width W}; the block's dictionary holds
  // npat x W offsets (pdict), prow one byte per row (pattern id; blocks are
  // strided by 256 bytes). The kernel reads 8 B per entry + 1 B per row
  // instead of 12 B per entry; the entries and their order are the CSR's, so
  // row sums are bitwise equal. pat == 0: none.
  int pat = 0;
  DVec<int> pdict, pmeta;
  DVec<unsigned char> prow;
  // x-window plan (spmv_prepare; irregular medium-row operators, e.g. the
  // coarse AMG levels): row blocks of <= 256 rows / 2048 entries whose
  // columns fall into <= kXtLines 128-byte lines of x. A block's lines are
  // bulk-copied into shared memory as runs of consecutive lines (xt_runs:
  // 32 {first line, line count} slots per block, xt_meta per block: {0, tail
  // slot or -1 or -2 = no window}); entries address the window through 16-bit local columns
  // (xt_col: slot * 16 + col % 16, same order as col). The row sums run
  // entirely out of shared memory: no scattered L1 gathers, 10 B per entry.
  // xt_nblk == 0: none. xt_plan: nblk+1 first rows, nblk+1 first entries.
  int xt_nblk = 0;
  // a built plan the per-matrix timing did not rule out; the hierarchy's
  // in-situ pass (MgrHier::tune_spmv) switches xt_nblk between 0 and this by
  // timing whole preconditioner applications
  int xt_plan_nblk = 0;
  int xt_geom = 0;  // 0: 256 rows / 2048 entries / 120 lines x 2 stages; 1: 128 / 1024 / 88 x 2 stages; 2: geometry 0's blocks x 3 stages
  DVec<int> xt_plan, xt_runs, xt_meta;
  DVec<unsigned short> xt_col;
  // Plan entries of the first block of every CTA (host copies, passed to the
  // staged / x-window kernels as launch parameters so that a CTA's first copy
  // is issued without a global-memory round trip): 8 ints per block
  // {r0, r1, p0, p1, d0, d1, w, tail}.
  std::vector<int> head, xt_head;
  // Team-sum SpMV of the tolerance-level solve (k_spmv_vec; lanes per row,
  // chosen per matrix by the setup timing). 0: none. Only consulted while a
  // TeamSums scope is active (the default solve); the bitwise paths never
  // take it.
  int vec = 0;
  // Team-sum BSR(3) copy (tolerance-level solve only; matrices whose block
  // rows hold full aligned 3 x 3 blocks, e.g. the elasticity displacement
  // operator): per block row the block columns (tcol) and the values as nine
  // planes of nb doubles (value k of block b at 9 * tptr[R] + k * nb + b), so
  // a warp reads each plane coalesced; 8.4 B per entry instead of 12.
  // tb == 0: none.
  int tb = 0;
  DVec<int> tptr, tcol;
  DVec<double> tval;
  bool empty() const { return rows == 0; }
};

// Scope in which SpMVs may sum a row in team order (fused multiply-adds per
// lane, shuffle tree) instead of the reference's left-to-right order: the
// default solve (tolerance-level parity, like its orthogonalisation). Thread-
// local, nestable; `on == false` leaves the current state.
struct TeamSums {
  // on: enable for the scope; off: disable for the scope (a bitwise
  // application inside a tolerance-level caller); neither: leave as is
  explicit TeamSums(bool on, bool off = false);
  ~TeamSums();
  TeamSums(const TeamSums&) = delete;
  TeamSums& operator=(const TeamSums&) = delete;
  static bool active();

 private:
  bool prev_;
};

// ---- primitives -----------------------------------------------------------
// Exclusive scan of n ints into out (out has n+1 entries, out[n] = total);
// returns the total (synchronizes).
int64_t exclusive_scan(const int* in, int* out, int n, cudaStream_t s);
int64_t exclusive_scan64(const int64_t* in, int64_t* out, int n, cudaStream_t s);
// Compact the indices i in [0,n) with flag[i] != 0 (ascending) into out;
// returns the count (synchronizes).
int select_flagged(const uint8_t* flag, int n, DVec<int>& out, cudaStream_t s);

// ---- construction / validation --------------------------------------------
// Upload host CSR and validate it like proj/src/sparse.cpp:24-41.
DCsr csr_from_host(int rows, int cols, const int* ptr, const int* col, const double* val,
                   cudaStream_t s);
DCsr csr_from_device(int rows, int cols, const int* ptr, const int* col, const double* val,
                     cudaStream_t s);
void csr_validate(const DCsr& A, cudaStream_t s);
DCsr csr_copy(const DCsr& A, cudaStream_t s);

// Evict the L2 by reading `bytes` of `buf` (clean lines; timing helpers).
void l2_flush_read(const void* buf, size_t bytes, cudaStream_t s);

// ---- SpMV family (solve path) ---------------------------------------------
// Build the block plan of the bulk-copy-staged SpMV for a solve-path matrix
// (rows >= 2048; kept only where it times faster than the direct kernels);
// matrices without a plan use the direct kernels. Host-
// synchronising: call at setup, never inside a captured region.
void spmv_prepare(DCsr& A, cudaStream_t s);
// Drop an x-window plan that the in-situ pass switched off.
void spmv_drop_xtile(DCsr& A);
// y = A x                                (Eigen y = A*x: 0 + row sum)
void spmv(const DCsr& A, const double* x, double* y, cudaStream_t s);
// y = b - A x ; if brow != null, b is gathered: b[brow[r]]
void spmv_residual(const DCsr& A, const double* x, const double* b, const int* brow, double* y,
                   cudaStream_t s);
// y += A x                               (Eigen y += A*x)
void spmv_add(const DCsr& A, const double* x, double* y, cudaStream_t s);
// z[r] = zprev(r) + (A e)[r], zprev(r) = fpos[r] >= 0 ? 0 + zF[fpos[r]] : 0
// (MGR prolongation, proj/src/mgr.cpp:210-217)
void spmv_prolong(const DCsr& P, const double* e, const int* fpos, const double* zF, double* z,
                  cudaStream_t s);
// MGR prolongation in split form: F rows of P as a column-major ELL of
// width w <= 4 (indexed by F position, so zF is read contiguously), C rows
// as their single identity entry; one launch covers both. Same arithmetic
// as spmv_prolong (row sums left to right, z = (0 + zF) + sum, C rows
// 0 + (0 + 1*e)). w == 0: P does not have that shape (use spmv_prolong).
struct ProlongPlan {
  int nf = 0, nc = 0, w = 0;
  const int* F = nullptr;  // level F / C lists (owned by the MGR level)
  const int* C = nullptr;
  DVec<int> ecol, ccol;
  DVec<double> eval, cval;
};
void prolong_prepare(const DCsr& P, const int* F, int nf, const int* C, int nc, ProlongPlan& out, cudaStream_t s);
void spmv_prolong_split(const ProlongPlan& pl, const double* e, const double* zF, double* z, cudaStream_t s);
// Jacobi correction sweep: znew = zold + w*(dinv*(b - A zold)), b gathered via brow.
void spmv_jacobi(const DCsr& A, const double* zold, const double* b, const int* brow,
                 const double* dinv, double w, double* znew, cudaStream_t s);
// Generalised sweep: zold == nullptr starts from the zero-guess iterate
// w*(dinv*b) computed on the fly (fusing the first sweep into this one);
// zacc != nullptr accumulates the result into zacc (fusing apply_add).
// Residual / plain product that also write the zero-start Jacobi iterate of
// their output, z0 = w * (dinv * y) (a fused k_jacobi0).
void spmv_residual_j0(const DCsr& A, const double* x, const double* b, double* y, const double* dinv, double w,
                      double* z0, cudaStream_t s);
void spmv_j0(const DCsr& A, const double* x, double* y, const double* dinv, double w, double* z0, cudaStream_t s);
void spmv_jacobi_ex(const DCsr& A, const double* zold, const double* b, const int* brow, const double* dinv,
                    double w, double* znew, double* zacc, cudaStream_t s);

// ---- setup kernels (bit-exact) --------------------------------------------
DCsr extract(const DCsr& A, const int* rows, int nrows, const int* cols, int ncols, cudaStream_t s);
DCsr transpose(const DCsr& A, cudaStream_t s);
// Eigen conservative product A*B.
DCsr spgemm(const DCsr& A, const DCsr& B, cudaStream_t s);
// Rows `rows` of A as a new CSR (used for injection R*(AP) = rows C of AP).
DCsr gather_rows(const DCsr& A, const int* rows, int nrows, cudaStream_t s);
// 1/a_ii with the reference's row-named errors (proj/src/sparse.cpp:87-104).
void diag_inverse(const DCsr& A, DVec<double>& dinv, cudaStream_t s);
// L1 diagonal with singleton (l1 = true) or whole-matrix range (l1 = false:
// d_i = sum of stored diagonal entries), proj/src/relax.cpp:34-48.
void l1_diagonal(const DCsr& A, bool singleton_ranges, DVec<double>& d, cudaStream_t s,
                 const int* owner = nullptr);
bool structurally_diagonal(const DCsr& A, cudaStream_t s);

// Host copies (tests / dumps).
struct HostCsr {
  int rows = 0, cols = 0;
  std::vector<int> ptr, col;
  std::vector<double> val;
};
HostCsr to_host(const DCsr& A, cudaStream_t s);

}  // namespace mgrx
