// Single-CTA dense LU with partial pivoting and its triangular solves. The
// pivot is the first row of maximal |a_ik| (Eigen maxCoeff semantics).
#include <algorithm>
#include <climits>
#include <numeric>

#include "dense.cuh"

namespace mgrx {
namespace {

constexpr int kT = 1024;

__global__ void k_densify(int n, const int* __restrict__ ptr, const int* __restrict__ col,
                          const double* __restrict__ val, double* __restrict__ M) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int k = ptr[i]; k < ptr[i + 1]; ++k) M[static_cast<size_t>(col[k]) * n + i] = val[k];
}

__global__ void __launch_bounds__(kT) k_lu(int n, double* M, int* perm, double tol, int* bad) {
  __shared__ double sv[kT];
  __shared__ int si[kT];
  __shared__ int piv;
  for (int i = threadIdx.x; i < n; i += kT) perm[i] = i;
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    double best = -1.0;
    int bi = n;
    for (int i = k + threadIdx.x; i < n; i += kT) {
      const double a = fabs(M[static_cast<size_t>(k) * n + i]);
      if (a > best || (a == best && i < bi)) {
        best = a;
        bi = i;
      }
    }
    sv[threadIdx.x] = best;
    si[threadIdx.x] = bi;
    __syncthreads();
    for (int w = kT / 2; w > 0; w >>= 1) {
      if (threadIdx.x < w) {
        const double a = sv[threadIdx.x + w];
        const int ai = si[threadIdx.x + w];
        if (a > sv[threadIdx.x] || (a == sv[threadIdx.x] && ai < si[threadIdx.x])) {
          sv[threadIdx.x] = a;
          si[threadIdx.x] = ai;
        }
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) piv = si[0];
    __syncthreads();
    const int p = piv;
    if (p != k) {
      for (int j = threadIdx.x; j < n; j += kT) {
        const size_t a = static_cast<size_t>(j) * n;
        const double t = M[a + k];
        M[a + k] = M[a + p];
        M[a + p] = t;
      }
      if (threadIdx.x == 0) {
        const int t = perm[k];
        perm[k] = perm[p];
        perm[p] = t;
      }
    }
    __syncthreads();
    const double pv = M[static_cast<size_t>(k) * n + k];
    if (pv != 0.0)
      for (int i = k + 1 + threadIdx.x; i < n; i += kT)
        M[static_cast<size_t>(k) * n + i] = __ddiv_rn(M[static_cast<size_t>(k) * n + i], pv);
    __syncthreads();
    const int m = n - k - 1;
    for (int t = threadIdx.x; t < m * m; t += kT) {
      const int jj = k + 1 + t / m, ii = k + 1 + t % m;
      const double ukj = M[static_cast<size_t>(jj) * n + k];
      if (ukj != 0.0)
        M[static_cast<size_t>(jj) * n + ii] =
            __dsub_rn(M[static_cast<size_t>(jj) * n + ii], __dmul_rn(M[static_cast<size_t>(k) * n + ii], ukj));
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    int b = -1;
    for (int i = 0; i < n; ++i)
      if (fabs(M[static_cast<size_t>(i) * n + i]) < tol) {
        b = i;
        break;
      }
    *bad = b;
  }
}

__global__ void __launch_bounds__(kT) k_lu_solve(int n, const double* __restrict__ M,
                                                 const int* __restrict__ perm,
                                                 const double* __restrict__ b, double* __restrict__ x) {
  pdl_enter();
  extern __shared__ double xs[];
  for (int i = threadIdx.x; i < n; i += kT) xs[i] = b[perm[i]];
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    const double xj = xs[j];
    for (int i = j + 1 + threadIdx.x; i < n; i += kT)
      xs[i] = __dsub_rn(xs[i], __dmul_rn(M[static_cast<size_t>(j) * n + i], xj));
    __syncthreads();
  }
  for (int j = n - 1; j >= 0; --j) {
    if (threadIdx.x == 0) xs[j] = __ddiv_rn(xs[j], M[static_cast<size_t>(j) * n + j]);
    __syncthreads();
    const double xj = xs[j];
    for (int i = threadIdx.x; i < j; i += kT)
      xs[i] = __dsub_rn(xs[i], __dmul_rn(M[static_cast<size_t>(j) * n + i], xj));
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += kT) x[i] = xs[i];
}

// Small systems (n <= 160, the usual coarsest AMG level): one warp, the
// factors staged in shared memory, lane l owning x_{l+32r} in registers, and
// the same update order as k_lu_solve (so results are bitwise identical) with
// warp shuffles in place of block barriers.
constexpr int kWarpLuMax = 160;
constexpr int kWarpLuR = (kWarpLuMax + 31) / 32;

__global__ void __launch_bounds__(32) k_lu_solve_warp(int n, const double* __restrict__ M,
                                                      const int* __restrict__ perm, const double* __restrict__ b,
                                                      double* __restrict__ x) {
  pdl_enter();
  extern __shared__ double Ms[];
  const int l = threadIdx.x;
  for (int e = l; e < n * n; e += 32) Ms[e] = M[e];
  double xr[kWarpLuR];
#pragma unroll
  for (int r = 0; r < kWarpLuR; ++r) {
    const int i = l + 32 * r;
    xr[r] = i < n ? b[perm[i]] : 0.0;
  }
  __syncwarp();
  // j = 32*jr + jl; x_j lives in register jr of lane jl (static index)
#pragma unroll
  for (int jr = 0; jr < kWarpLuR; ++jr) {
    for (int jl = 0; jl < 32; ++jl) {
      const int j = 32 * jr + jl;
      if (j >= n) break;
      const double xj = __shfl_sync(0xffffffffu, xr[jr], jl);
      const double* Mj = Ms + j * n;
#pragma unroll
      for (int r = 0; r < kWarpLuR; ++r) {
        const int i = l + 32 * r;
        if (i > j && i < n) xr[r] = __dsub_rn(xr[r], __dmul_rn(Mj[i], xj));
      }
    }
  }
#pragma unroll
  for (int jr = kWarpLuR - 1; jr >= 0; --jr) {
    for (int jl = 31; jl >= 0; --jl) {
      const int j = 32 * jr + jl;
      if (j >= n) continue;
      const double* Mj = Ms + j * n;
      if (l == jl) xr[jr] = __ddiv_rn(xr[jr], Mj[j]);
      const double xj = __shfl_sync(0xffffffffu, xr[jr], jl);
#pragma unroll
      for (int r = 0; r < kWarpLuR; ++r) {
        const int i = l + 32 * r;
        if (i < j) xr[r] = __dsub_rn(xr[r], __dmul_rn(Mj[i], xj));
      }
    }
  }
#pragma unroll
  for (int r = 0; r < kWarpLuR; ++r) {
    const int i = l + 32 * r;
    if (i < n) x[i] = xr[r];
  }
}

// ---- per-component (block-diagonal) factorization and solve ---------------
// Block b: rows rows[bst[b] .. bst[b+1]) (ascending), factors column-major at
// blu + boff[b]. One CTA per block for the factorization (the k_lu algorithm
// on the block), one warp per block for the solve.
__global__ void k_densify_blocks(int nb, const int* __restrict__ bst, const long long* __restrict__ boff,
                                 const int* __restrict__ rows, const int* __restrict__ lpos,
                                 const int* __restrict__ ptr, const int* __restrict__ col,
                                 const double* __restrict__ val, double* __restrict__ blu) {
  const int b = blockIdx.x;
  const int lo = bst[b], s = bst[b + 1] - lo;
  double* M = blu + boff[b];
  for (long long e = threadIdx.x; e < static_cast<long long>(s) * s; e += blockDim.x) M[e] = 0.0;
  __syncthreads();
  for (int i = threadIdx.x; i < s; i += blockDim.x) {
    const int g = rows[lo + i];
    for (int k = ptr[g]; k < ptr[g + 1]; ++k) M[static_cast<size_t>(lpos[col[k]]) * s + i] = val[k];
  }
}

__global__ void __launch_bounds__(kT) k_lu_blocks(const int* __restrict__ bst, const long long* __restrict__ boff,
                                                  const int* __restrict__ rows, double* blu, int* perm, double tol,
                                                  int* bad) {
  __shared__ double sv[kT];
  __shared__ int si[kT];
  __shared__ int piv;
  const int b = blockIdx.x;
  const int lo = bst[b], n = bst[b + 1] - lo;
  double* M = blu + boff[b];
  int* pm = perm + lo;
  for (int i = threadIdx.x; i < n; i += kT) pm[i] = i;
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    double best = -1.0;
    int bi = n;
    for (int i = k + threadIdx.x; i < n; i += kT) {
      const double a = fabs(M[static_cast<size_t>(k) * n + i]);
      if (a > best || (a == best && i < bi)) {
        best = a;
        bi = i;
      }
    }
    sv[threadIdx.x] = best;
    si[threadIdx.x] = bi;
    __syncthreads();
    for (int w = kT / 2; w > 0; w >>= 1) {
      if (threadIdx.x < w) {
        const double a = sv[threadIdx.x + w];
        const int ai = si[threadIdx.x + w];
        if (a > sv[threadIdx.x] || (a == sv[threadIdx.x] && ai < si[threadIdx.x])) {
          sv[threadIdx.x] = a;
          si[threadIdx.x] = ai;
        }
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) piv = si[0];
    __syncthreads();
    const int p = piv;
    if (p != k) {
      for (int j = threadIdx.x; j < n; j += kT) {
        const size_t a = static_cast<size_t>(j) * n;
        const double t = M[a + k];
        M[a + k] = M[a + p];
        M[a + p] = t;
      }
      if (threadIdx.x == 0) {
        const int t = pm[k];
        pm[k] = pm[p];
        pm[p] = t;
      }
    }
    __syncthreads();
    const double pv = M[static_cast<size_t>(k) * n + k];
    if (pv != 0.0)
      for (int i = k + 1 + threadIdx.x; i < n; i += kT)
        M[static_cast<size_t>(k) * n + i] = __ddiv_rn(M[static_cast<size_t>(k) * n + i], pv);
    __syncthreads();
    const int m = n - k - 1;
    for (int t = threadIdx.x; t < m * m; t += kT) {
      const int jj = k + 1 + t / m, ii = k + 1 + t % m;
      const double ukj = M[static_cast<size_t>(jj) * n + k];
      if (ukj != 0.0)
        M[static_cast<size_t>(jj) * n + ii] =
            __dsub_rn(M[static_cast<size_t>(jj) * n + ii], __dmul_rn(M[static_cast<size_t>(k) * n + ii], ukj));
    }
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int i = 0; i < n; ++i)
      if (fabs(M[static_cast<size_t>(i) * n + i]) < tol) {
        atomicMin(bad, rows[lo + i]);
        break;
      }
}

// Triangular solves of one block per CTA, panel-blocked: kW columns at a
// time, warp 0 runs the panel's triangle with the lane-owned iterate in
// registers (its row entries preloaded), then all threads apply the panel's
// columns to the remaining rows. Every x_i still receives its updates in the
// unblocked order (j ascending forward, descending backward, the division
// by u_ii right after the last update from j > i), so results are bitwise
// those of k_lu_solve / DenseLU::solve. rows == nullptr: identity row map.
// kStage: the panels' columns (contiguous in the column-major factors) are
// staged in shared memory with cp.async, double-buffered one panel ahead, so
// the triangle and the update read shared memory instead of paying an L2 /
// HBM round trip per panel.
constexpr int kPT = 256;
__device__ __forceinline__ void cpa8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cpa_commit_group() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int kW, bool kStage>
__global__ void __launch_bounds__(kPT) k_lu_solve_panel(const int* __restrict__ bst, const long long* __restrict__ boff,
                                                        const int* __restrict__ rows, const double* __restrict__ blu,
                                                        const int* __restrict__ perm, int n1,
                                                        const double* __restrict__ bvec, double* __restrict__ x) {
  pdl_enter();
  extern __shared__ double sh[];
  const int b = blockIdx.x;
  const int lo = bst ? bst[b] : 0;
  const int n = bst ? bst[b + 1] - lo : n1;
  const double* M = blu + (boff ? boff[b] : 0);
  const int* pm = perm + lo;
  const int T = threadIdx.x, l = T & 31;
  double* xs = sh;
  double* pbuf = sh + ((n + 1) & ~1);  // two panel buffers of kW * n
  auto stage = [&](int j0, int jn, int slot) {
    if (kStage) {
      const double* src = M + static_cast<size_t>(j0) * n;
      double* dst = pbuf + static_cast<size_t>(slot) * kW * n;
      for (int e = T; e < jn * n; e += kPT) cpa8(dst + e, src + e);
      cpa_commit_group();
    }
  };
  auto panel = [&](int j0, int slot) -> const double* {
    return kStage ? pbuf + static_cast<size_t>(slot) * kW * n : M + static_cast<size_t>(j0) * n;
  };
  for (int i = T; i < n; i += kPT) xs[i] = bvec[rows ? rows[lo + pm[i]] : pm[i]];
  const int np = (n + kW - 1) / kW;
  // forward: unit lower triangle
  stage(0, n < kW ? n : kW, 0);
  for (int p = 0; p < np; ++p) {
    const int j0 = p * kW, jn = min(kW, n - j0);
    if (kStage) cpa_wait_group<0>();  // panel p (issued one panel ago) has landed
    __syncthreads();                   // ... for every thread; panel p-1's readers are done
    if (p + 1 < np) stage(j0 + kW, min(kW, n - j0 - kW), (p + 1) & 1);
    const double* P = panel(j0, p & 1);  // P[jj * n + i] = M(i, j0 + jj)
    if (T < 32) {
      const int i = j0 + l;
      double m[kW];
#pragma unroll
      for (int jj = 0; jj < kW; ++jj) m[jj] = (jj < l && l < jn) ? P[jj * n + i] : 0.0;
      double xv = l < jn ? xs[i] : 0.0;
#pragma unroll
      for (int jj = 0; jj < kW; ++jj) {
        const double xj = __shfl_sync(0xffffffffu, xv, jj);
        if (jj < l && l < jn) xv = __dsub_rn(xv, __dmul_rn(m[jj], xj));
      }
      if (l < jn) xs[i] = xv;
    }
    __syncthreads();
    for (int i = j0 + jn + T; i < n; i += kPT) {
      double v = xs[i];
      for (int jj = 0; jj < jn; ++jj) v = __dsub_rn(v, __dmul_rn(P[jj * n + i], xs[j0 + jj]));
      xs[i] = v;
    }
  }
  __syncthreads();
  // backward: upper triangle, division before the updates of each column
  {
    const int j0f = (np - 1) * kW;
    stage(j0f, n - j0f, 0);
  }
  for (int p = np - 1, it = 0; p >= 0; --p, ++it) {
    const int j0 = p * kW, jn = min(kW, n - j0);
    if (kStage) cpa_wait_group<0>();
    __syncthreads();
    if (p > 0) stage(j0 - kW, kW, (it + 1) & 1);
    const double* P = panel(j0, it & 1);
    if (T < 32) {
      const int i = j0 + l;
      double m[kW];
#pragma unroll
      for (int jj = 0; jj < kW; ++jj) m[jj] = (jj >= l && jj < jn && l < jn) ? P[jj * n + i] : 1.0;
      double xv = l < jn ? xs[i] : 0.0;
#pragma unroll
      for (int jj = kW - 1; jj >= 0; --jj) {
        if (jj < jn) {
          if (l == jj) xv = __ddiv_rn(xv, m[jj]);
          const double xj = __shfl_sync(0xffffffffu, xv, jj);
          if (l < jj) xv = __dsub_rn(xv, __dmul_rn(m[jj], xj));
        }
      }
      if (l < jn) xs[i] = xv;
    }
    __syncthreads();
    for (int i = T; i < j0; i += kPT) {
      double v = xs[i];
      for (int jj = jn - 1; jj >= 0; --jj) v = __dsub_rn(v, __dmul_rn(P[jj * n + i], xs[j0 + jj]));
      xs[i] = v;
    }
  }
  __syncthreads();
  for (int i = T; i < n; i += kPT) x[rows ? rows[lo + i] : i] = xs[i];
}

// The panel solve variant for blocks of up to n rows: the widest panel whose
// double buffer fits in shared memory. prepare (at factorization, outside
// any graph capture) raises the kernel's shared-memory limit.
using PanelKern = void (*)(const int*, const long long*, const int*, const double*, const int*, int, const double*,
                           double*);
PanelKern panel_variant(int n, size_t& sm) {
  const size_t xs = sizeof(double) * ((n + 1) & ~1);
  auto smem = [&](int w) { return xs + 2 * sizeof(double) * w * static_cast<size_t>(n); };
  constexpr size_t kMax = 200 * 1024;
  PanelKern k = k_lu_solve_panel<32, false>;
  sm = xs;
  if (smem(8) <= kMax) {
    k = k_lu_solve_panel<8, true>;
    sm = smem(8);
  }
  if (smem(16) <= kMax) {
    k = k_lu_solve_panel<16, true>;
    sm = smem(16);
  }
  if (smem(32) <= kMax) {
    k = k_lu_solve_panel<32, true>;
    sm = smem(32);
  }
  return k;
}
void prepare_panel_solve(int n) {
  size_t sm = 0;
  PanelKern k = panel_variant(n, sm);
  if (sm > 48 * 1024)
    ensure_smem(reinterpret_cast<const void*>(k), static_cast<size_t>(static_cast<int>(sm)));
}
void launch_panel_solve(int grid, int n, const int* bst, const long long* boff, const int* rows, const double* lu,
                        const int* perm, int n1, const double* b, double* x, cudaStream_t s) {
  size_t sm = 0;
  PanelKern k = panel_variant(n, sm);
  launch_pdl(k, grid, kPT, sm, s, bst, boff, rows, lu, perm, n1, b, x);
  MGRX_LAUNCH_CK();
  count_launch();
}

// ---------------------------------------------------------------------------
// Cluster-parallel triangular solves for blocks of <= 256 rows (the MGR
// coarse well blocks of the compositional strategy, 250 rows each; small
// AMG coarsest grids). The single-CTA panel solve streams the whole n x n
// factor through one SM twice per solve (cfg3: 96 us of an 856 us GMRES
// step). Here block b is solved by a thread-block cluster of C = ceil(n/32)
// CTAs: CTA c owns rows 32c..32c+31 (one warp, one lane per row) and holds
// those rows of L and U in shared memory (its "slab", re-laid out at
// factorization time, one bulk copy per solve). Forward: CTA c applies the
// panels of the CTAs before it as their solved values arrive, in panel
// order and column order within a panel, then runs its own panel triangle
// and stores its 32 values into the shared memory of every later CTA of the
// cluster (DSMEM) behind a per-panel flag. Backward mirrors it. Every x_i
// receives exactly the updates of the unblocked algorithm in the same order
// (the panel solve's k_lu_solve_panel bodies), so results are bitwise equal.
constexpr int kClMax = 8;  // CTAs per cluster (portable limit) -> blocks of <= 256 rows

// slab[((b * C + c) * ns + j) * 32 + r] = M_b(32c + r, j) (0 outside the block)
__global__ void k_slabify(int nb, int C, int ns, const int* __restrict__ bst, const long long* __restrict__ boff,
                          int n1, const double* __restrict__ blu, double* __restrict__ slab) {
  const long long total = static_cast<long long>(nb) * C * ns * 32;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(e & 31);
    const long long q = e >> 5;
    const int j = static_cast<int>(q % ns);
    const long long bc = q / ns;
    const int c = static_cast<int>(bc % C), b = static_cast<int>(bc / C);
    const int n = bst ? bst[b + 1] - bst[b] : n1;
    const int i = 32 * c + r;
    const double* M = blu + (boff ? boff[b] : 0);
    slab[e] = (i < n && j < n) ? M[static_cast<size_t>(j) * n + i] : 0.0;
  }
}

__device__ __forceinline__ unsigned cl_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cl_map(const void* p, unsigned cta) {
  unsigned a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
               : "=r"(a)
               : "r"(static_cast<unsigned>(__cvta_generic_to_shared(p))), "r"(cta));
  return a;
}
__device__ __forceinline__ void cl_st_f64(unsigned a, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void cl_st_u32(unsigned a, unsigned v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

__global__ void __launch_bounds__(32) k_lu_solve_cluster(int ns, const int* __restrict__ bst,
                                                         const int* __restrict__ rows,
                                                         const double* __restrict__ slab,
                                                         const int* __restrict__ perm, int n1,
                                                         const double* __restrict__ bvec, double* __restrict__ x) {
  pdl_enter();
  extern __shared__ __align__(16) double csm[];
  double* S = csm;                 // [ns][32] this CTA's rows of L and U
  double* xf = csm + ns * 32;      // solved values of the other CTAs' rows
  __shared__ volatile unsigned flag[2][kClMax];
  __shared__ __align__(8) unsigned long long mbar;
  const unsigned c = cl_rank();
  unsigned nc;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(nc));
  const int b = blockIdx.x / nc;
  const int l = threadIdx.x;
  const int lo = bst ? bst[b] : 0;
  const int n = bst ? bst[b + 1] - lo : n1;
  const int* pm = perm + lo;
  const int r0 = 32 * c;
  const int np = (n + 31) / 32;  // panels = active CTAs of this block
  if (l < 2 * kClMax) flag[l / kClMax][l % kClMax] = 0u;
  const unsigned mb = static_cast<unsigned>(__cvta_generic_to_shared(&mbar));
  if (l == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(mb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cl_sync();  // flags initialised cluster-wide before any remote store
  const bool active = r0 < n;
  if (active) {
    const unsigned bytes = static_cast<unsigned>(ns) * 32u * 8u;
    if (l == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              static_cast<unsigned>(__cvta_generic_to_shared(S))),
          "l"(slab + (static_cast<size_t>(blockIdx.x) * ns) * 32), "r"(bytes), "r"(mb)
          : "memory");
    }
    const int i = r0 + l;
    const int jn_own = min(32, n - r0);
    double xv = l < jn_own ? bvec[rows ? rows[lo + pm[i]] : pm[i]] : 0.0;
    unsigned done = 0;
    do {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done)
                   : "r"(mb), "r"(0u)
                   : "memory");
    } while (!done);
    // forward: panels of the earlier CTAs, in order, as they arrive
    for (int p = 0; p < static_cast<int>(c); ++p) {
      while (flag[0][p] == 0u) {
      }
      asm volatile("fence.acq_rel.cluster;" ::: "memory");
      const int j0 = 32 * p, jn = min(32, n - j0);
      for (int jj = 0; jj < jn; ++jj) xv = __dsub_rn(xv, __dmul_rn(S[(j0 + jj) * 32 + l], xf[j0 + jj]));
    }
    // own panel triangle (unit lower)
    {
      double m[32];
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) m[jj] = (jj < l && l < jn_own) ? S[(r0 + jj) * 32 + l] : 0.0;
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) {
        const double xj = __shfl_sync(0xffffffffu, xv, jj);
        if (jj < l && l < jn_own) xv = __dsub_rn(xv, __dmul_rn(m[jj], xj));
      }
    }
    // publish to the later CTAs of the block
    for (int q = static_cast<int>(c) + 1; q < np; ++q) {
      if (l < jn_own) cl_st_f64(cl_map(xf + i, q), xv);
      __syncwarp();
      if (l == 0) {
        asm volatile("fence.acq_rel.cluster;" ::: "memory");
        cl_st_u32(cl_map(const_cast<unsigned*>(&flag[0][c]), q), 1u);
      }
    }
    // backward: panels of the later CTAs, last first
    for (int p = np - 1; p > static_cast<int>(c); --p) {
      while (flag[1][p] == 0u) {
      }
      asm volatile("fence.acq_rel.cluster;" ::: "memory");
      const int j0 = 32 * p, jn = min(32, n - j0);
      for (int jj = jn - 1; jj >= 0; --jj) xv = __dsub_rn(xv, __dmul_rn(S[(j0 + jj) * 32 + l], xf[j0 + jj]));
    }
    // own panel triangle (upper, division before the column's updates)
    {
      double m[32];
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) m[jj] = (jj >= l && jj < jn_own && l < jn_own) ? S[(r0 + jj) * 32 + l] : 1.0;
#pragma unroll
      for (int jj = 31; jj >= 0; --jj) {
        if (jj < jn_own) {
          if (l == jj) xv = __ddiv_rn(xv, m[jj]);
          const double xj = __shfl_sync(0xffffffffu, xv, jj);
          if (l < jj) xv = __dsub_rn(xv, __dmul_rn(m[jj], xj));
        }
      }
    }
    for (int q = static_cast<int>(c) - 1; q >= 0; --q) {
      if (l < jn_own) cl_st_f64(cl_map(xf + i, q), xv);
      __syncwarp();
      if (l == 0) {
        asm volatile("fence.acq_rel.cluster;" ::: "memory");
        cl_st_u32(cl_map(const_cast<unsigned*>(&flag[1][c]), q), 1u);
      }
    }
    if (l < jn_own) x[rows ? rows[lo + i] : i] = xv;
  }
  cl_sync();  // no CTA leaves while a peer may still store into its shared memory
}

bool cluster_solve_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("MGRX_DENSE_CLUSTER");
    return !v || std::atoi(v) != 0;
  }();
  return on;
}

// Re-lay the factors out as per-CTA slabs (after factorization).
void build_slabs(DenseLU& f, cudaStream_t s) {
  f.ccl = 0;
  const int nmax = f.nb > 1 ? f.max_block : f.n;
  if (!cluster_solve_enabled() || nmax <= 0 || nmax > 32 * kClMax) return;
  const int C = (nmax + 31) / 32;
  const int ns = nmax;
  const size_t smem = sizeof(double) * (static_cast<size_t>(ns) * 32 + ns + 2);
  if (smem > 48 * 1024)
    ensure_smem(reinterpret_cast<const void*>(k_lu_solve_cluster), static_cast<size_t>(static_cast<int>(smem)));
  f.slab.alloc(static_cast<size_t>(f.nb) * C * ns * 32, s);
  const long long total = static_cast<long long>(f.nb) * C * ns * 32;
  const int grid = static_cast<int>(std::min<long long>((total + 255) / 256, 148 * 16));
  if (f.nb > 1)
    k_slabify<<<grid, 256, 0, s>>>(f.nb, C, ns, f.bst.get(), f.boff.get(), 0, f.blu.get(), f.slab.get());
  else
    k_slabify<<<grid, 256, 0, s>>>(1, C, ns, nullptr, nullptr, f.n, f.lu.get(), f.slab.get());
  MGRX_LAUNCH_CK();
  count_launch();
  f.ccl = C;
  f.slab_n = ns;
}

void launch_cluster_solve(const DenseLU& f, const double* b, double* x, cudaStream_t s) {
  const int C = f.ccl, ns = f.slab_n;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(f.nb * C);
  cfg.blockDim = dim3(32);
  cfg.dynamicSmemBytes = sizeof(double) * (static_cast<size_t>(ns) * 32 + ns + 2);
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = C;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  const int* bst = f.nb > 1 ? f.bst.get() : nullptr;
  const int* rows = f.nb > 1 ? f.rows.get() : nullptr;
  MGRX_CK(cudaLaunchKernelEx(&cfg, k_lu_solve_cluster, ns, bst, rows, static_cast<const double*>(f.slab.get()),
                             static_cast<const int*>(f.perm.get()), f.n, b, x));
  count_launch();
}

// Connected components of the symmetrised pattern of A (host; A is a
// coarse system): component lists ascending, components ordered by their
// smallest row.
std::vector<std::vector<int>> components(int n, const std::vector<int>& ptr, const std::vector<int>& col) {
  std::vector<int> par(n);
  std::iota(par.begin(), par.end(), 0);
  auto find = [&](int a) {
    while (par[a] != a) a = par[a] = par[par[a]];
    return a;
  };
  for (int i = 0; i < n; ++i)
    for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
      const int a = find(i), c = find(col[k]);
      if (a != c) par[std::max(a, c)] = std::min(a, c);
    }
  std::vector<int> id(n, -1);
  std::vector<std::vector<int>> out;
  for (int i = 0; i < n; ++i) {
    const int r = find(i);
    if (id[r] < 0) {
      id[r] = static_cast<int>(out.size());
      out.emplace_back();
    }
    out[id[r]].push_back(i);
  }
  return out;
}

}  // namespace

void dense_factor(const DCsr& A, DenseLU& out, cudaStream_t s, double pivot_tol, bool allow_blocks) {
  if (A.rows != A.cols) throw RuntimeError("dense LU: matrix not square");
  const int n = A.rows;
  out.n = n;
  out.nb = 1;
  // block-diagonal systems: factor per connected component
  if (n > 1 && allow_blocks) {
    const std::vector<int> ptr = A.ptr.download(n + 1);
    const std::vector<int> col = A.col.download(ptr[n]);
    const std::vector<std::vector<int>> comp = components(n, ptr, col);
    if (comp.size() > 1) {
      out.nb = static_cast<int>(comp.size());
      std::vector<int> rows, bst(1, 0), lpos(n);
      std::vector<long long> boff(1, 0);
      out.max_block = 0;
      for (const auto& c : comp) {
        for (size_t i = 0; i < c.size(); ++i) lpos[c[i]] = static_cast<int>(i);
        rows.insert(rows.end(), c.begin(), c.end());
        bst.push_back(static_cast<int>(rows.size()));
        boff.push_back(boff.back() + static_cast<long long>(c.size()) * c.size());
        out.max_block = std::max(out.max_block, static_cast<int>(c.size()));
      }
      if (out.max_block > 6000) throw RuntimeError("dense LU: block too large for the single-CTA factorization");
      out.rows.alloc(n, s);
      out.rows.upload(rows.data(), n);
      out.bst.alloc(out.nb + 1, s);
      out.bst.upload(bst.data(), out.nb + 1);
      out.boff.alloc(out.nb + 1, s);
      out.boff.upload(boff.data(), out.nb + 1);
      out.blu.alloc(boff.back(), s);
      out.perm.alloc(n, s);
      out.lu.alloc(1, s);
      DVec<int> dl(n, s);
      dl.upload(lpos.data(), n);
      k_densify_blocks<<<out.nb, 256, 0, s>>>(out.nb, out.bst.get(), out.boff.get(), out.rows.get(), dl.get(),
                                             A.ptr.get(), A.col.get(), A.val.get(), out.blu.get());
      DVec<int> bad(1, s);
      const int big = INT_MAX;
      bad.upload(&big, 1);
      k_lu_blocks<<<out.nb, kT, 0, s>>>(out.bst.get(), out.boff.get(), out.rows.get(), out.blu.get(),
                                        out.perm.get(), pivot_tol, bad.get());
      MGRX_LAUNCH_CK();
      count_launch(2);
      if (sizeof(double) * out.max_block > 200 * 1024)
        throw RuntimeError("dense LU solve: block too large for shared memory");
      prepare_panel_solve(out.max_block);
      build_slabs(out, s);
      const int b = read_scalar(bad.get(), s);
      // the dense algorithm reports the first singular pivot in row order
      if (b != INT_MAX) throw RuntimeError("dense LU: matrix numerically singular (pivot " + std::to_string(b) + ")");
      dense_build_inverse(out, s);
      return;
    }
  }
  if (n > 6000) throw RuntimeError("dense LU: matrix too large for the single-CTA factorization");
  out.lu.alloc(static_cast<size_t>(n) * n, s);
  out.perm.alloc(n > 0 ? n : 1, s);
  out.lu.zero();
  if (n == 0) return;
  k_densify<<<blocks_for(n, 256), 256, 0, s>>>(n, A.ptr.get(), A.col.get(), A.val.get(), out.lu.get());
  DVec<int> bad(1, s);
  k_lu<<<1, kT, 0, s>>>(n, out.lu.get(), out.perm.get(), pivot_tol, bad.get());
  MGRX_LAUNCH_CK();
  count_launch(2);
  if (n <= kWarpLuMax) {
    const int smw = static_cast<int>(sizeof(double) * n * n);
    if (smw > 48 * 1024)
      ensure_smem(reinterpret_cast<const void*>(k_lu_solve_warp), static_cast<size_t>(smw));
  }
  const size_t sm = sizeof(double) * n;
  if (sm > 200 * 1024) throw RuntimeError("dense LU solve: system too large for shared memory");
  if (sm > 48 * 1024)
    ensure_smem(reinterpret_cast<const void*>(k_lu_solve), static_cast<size_t>(static_cast<int>(sm)));
  prepare_panel_solve(n);
  build_slabs(out, s);
  const int b = read_scalar(bad.get(), s);
  if (b >= 0) throw RuntimeError("dense LU: matrix numerically singular (pivot " + std::to_string(b) + ")");
  dense_build_inverse(out, s);
}

namespace {
constexpr int kInvMax = 1024;   // rows per block for the explicit inverse
constexpr long long kInvEntries = 16ll << 20;

// Column j of block b's inverse = the LU solve of e_j (unit-lower forward,
// upper backward substitution), one warp per column, the column held in
// registers (lane l owns rows l, l+32, ...).
__global__ void __launch_bounds__(256) k_lu_inverse(int nb, int n1, const int* __restrict__ bst,
                                                    const long long* __restrict__ boff, const double* __restrict__ lu,
                                                    const int* __restrict__ perm_all,
                                                    const long long* __restrict__ ioff, double* __restrict__ inv) {
  constexpr int kQ = kInvMax / 32;
  const int b = blockIdx.y;
  const int s = nb > 1 ? bst[b + 1] - bst[b] : n1;
  const int j = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int l = threadIdx.x & 31;
  if (j >= s) return;
  const double* LU = lu + (nb > 1 ? boff[b] : 0);
  const int* perm = perm_all + (nb > 1 ? bst[b] : 0);
  double y[kQ];
#pragma unroll
  for (int q = 0; q < kQ; ++q) {
    const int i = l + 32 * q;
    y[q] = (i < s && perm[i] == j) ? 1.0 : 0.0;
  }
  for (int k = 0; k < s; ++k) {  // L y = P e_j
    double v = 0.0;
#pragma unroll
    for (int q = 0; q < kQ; ++q)
      if (q == (k >> 5)) v = y[q];
    const double yk = __shfl_sync(0xffffffffu, v, k & 31);
    const double* col = LU + static_cast<size_t>(k) * s;
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
      const int i = l + 32 * q;
      if (i > k && i < s) y[q] = fma(-col[i], yk, y[q]);
    }
  }
  for (int k = s - 1; k >= 0; --k) {  // U x = y
    const double* col = LU + static_cast<size_t>(k) * s;
    double v = 0.0;
#pragma unroll
    for (int q = 0; q < kQ; ++q)
      if (q == (k >> 5)) v = y[q];
    const double xk = __shfl_sync(0xffffffffu, v, k & 31) / col[k];
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
      const int i = l + 32 * q;
      if (i == k) y[q] = xk;
      else if (i < k) y[q] = fma(-col[i], xk, y[q]);
    }
  }
  double* out = inv + ioff[b];
#pragma unroll
  for (int q = 0; q < kQ; ++q) {
    const int i = l + 32 * q;
    if (i < s) out[static_cast<size_t>(i) * s + j] = y[q];
  }
}

// x[rows[p]] = sum_j inv_b(i, j) b[rows[bst_b + j]], warp per position p.
__global__ void __launch_bounds__(256) k_inv_apply(int n, int nb, const int* __restrict__ bst,
                                                   const int* __restrict__ rows, const int* __restrict__ pblk,
                                                   const long long* __restrict__ ioff,
                                                   const double* __restrict__ inv, const double* __restrict__ bv,
                                                   double* __restrict__ x) {
  pdl_enter();
  const int p = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int l = threadIdx.x & 31;
  if (p >= n) return;
  const int b = nb > 1 ? pblk[p] : 0;
  const int b0 = nb > 1 ? bst[b] : 0;
  const int s = nb > 1 ? bst[b + 1] - b0 : n;
  const int i = p - b0;
  const double* row = inv + ioff[b] + static_cast<size_t>(i) * s;
  double acc = 0.0;
  for (int j = l; j < s; j += 32) acc = fma(__ldg(row + j), __ldg(bv + (rows ? __ldg(rows + b0 + j) : b0 + j)), acc);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (l == 0) x[rows ? rows[p] : p] = acc;
}
}  // namespace

void dense_build_inverse(DenseLU& f, cudaStream_t s) {
  f.has_inv = false;
  if (f.n <= 0) return;
  const int nb = f.nb;
  std::vector<int> bst(nb + 1, 0);
  if (nb > 1) bst = f.bst.download(nb + 1);
  else bst[1] = f.n;
  std::vector<long long> io(nb + 1, 0);
  std::vector<int> pb(f.n);
  int maxs = 0;
  for (int b = 0; b < nb; ++b) {
    const int sb = bst[b + 1] - bst[b];
    maxs = std::max(maxs, sb);
    io[b + 1] = io[b] + static_cast<long long>(sb) * sb;
    for (int p = bst[b]; p < bst[b + 1]; ++p) pb[p] = b;
  }
  if (maxs > kInvMax || io[nb] > kInvEntries) return;
  f.ioff.alloc(nb + 1, s);
  f.ioff.upload(io.data(), nb + 1);
  f.pblk.alloc(f.n, s);
  f.pblk.upload(pb.data(), f.n);
  f.inv.alloc(static_cast<size_t>(io[nb]), s);
  const dim3 grid((maxs + 7) / 8, nb);
  if (nb > 1)
    k_lu_inverse<<<grid, 256, 0, s>>>(nb, f.n, f.bst.get(), f.boff.get(), f.blu.get(), f.perm.get(), f.ioff.get(),
                                      f.inv.get());
  else
    k_lu_inverse<<<grid, 256, 0, s>>>(1, f.n, nullptr, nullptr, f.lu.get(), f.perm.get(), f.ioff.get(), f.inv.get());
  MGRX_LAUNCH_CK();
  count_launch();
  f.has_inv = true;
}

void dense_solve(const DenseLU& f, const double* b, double* x, cudaStream_t s, bool exact) {
  if (f.n == 0) return;
  if (!exact && f.has_inv) {
    launch_pdl(k_inv_apply, dim3((f.n + 7) / 8), dim3(256), 0, s, f.n, f.nb, f.nb > 1 ? f.bst.get() : nullptr,
               f.nb > 1 ? f.rows.get() : nullptr, f.nb > 1 ? f.pblk.get() : nullptr, f.ioff.get(), f.inv.get(), b, x);
    count_launch();
    return;
  }
  if (f.ccl > 0) {
    launch_cluster_solve(f, b, x, s);
    return;
  }
  if (f.nb > 1) {
    launch_panel_solve(f.nb, f.max_block, f.bst.get(), f.boff.get(), f.rows.get(), f.blu.get(), f.perm.get(), 0, b, x,
                       s);
    return;
  }
  // MGRX_DENSE_SOLVE=warp|cta: the earlier one-warp (factors in shared
  // memory) / one-CTA column-sweep kernels; default: the panel-blocked CTA
  // solve (all three bitwise identical)
  static const int mode = [] {
    const char* e = std::getenv("MGRX_DENSE_SOLVE");
    if (e && e[0] == 'w') return 1;
    if (e && e[0] == 'c') return 2;
    return 0;
  }();
  if (mode == 1 && f.n <= kWarpLuMax) {
    launch_pdl(k_lu_solve_warp, 1, 32, sizeof(double) * f.n * f.n, s, f.n, f.lu.get(), f.perm.get(), b, x);
    MGRX_LAUNCH_CK();
    count_launch();
    return;
  }
  const size_t sm = sizeof(double) * f.n;
  if (mode == 2) {
    launch_pdl(k_lu_solve, 1, kT, sm, s, f.n, f.lu.get(), f.perm.get(), b, x);
    MGRX_LAUNCH_CK();
    count_launch();
    return;
  }
  launch_panel_solve(1, f.n, nullptr, nullptr, nullptr, f.lu.get(), f.perm.get(), f.n, b, x, s);
}

}  // namespace mgrx
