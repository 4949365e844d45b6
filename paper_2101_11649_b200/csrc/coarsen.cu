// AMG coarsening kernels. Every decision uses the reference's exact
// comparisons (std::max as (a < b) ? b : a, strict/non-strict tests as in
// proj/src/amg.cpp) on bit-identical operands, so C/F splittings and P
// patterns/values match the CPU oracle bit for bit.
#include "coarsen.cuh"

namespace mgrx {
namespace {

__device__ __forceinline__ double stdmax(double a, double b) { return (a < b) ? b : a; }

// ---- strength (amg.cpp:11-34) -----------------------------------------------
template <bool kFill>
__global__ void k_strength(int n, double theta, const int* __restrict__ ptr,
                           const int* __restrict__ col, const double* __restrict__ val,
                           int* __restrict__ cnt, const int* __restrict__ optr,
                           int* __restrict__ ocol, double* __restrict__ oval) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double mneg = 0.0, mabs = 0.0;
  for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
    if (col[k] == i) continue;
    mneg = stdmax(mneg, -val[k]);
    mabs = stdmax(mabs, fabs(val[k]));
  }
  int c = 0;
  int o = kFill ? optr[i] : 0;
  if (mabs != 0.0) {
    const bool neg = mneg > 0.0;
    const double cut = __dmul_rn(theta, neg ? mneg : mabs);
    for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
      if (col[k] == i) continue;
      const double m = neg ? -val[k] : fabs(val[k]);
      if (m >= cut && m > 0.0) {
        if (kFill) {
          ocol[o] = col[k];
          oval[o] = 1.0;
          ++o;
        }
        ++c;
      }
    }
  }
  if (!kFill) cnt[i] = c;
}

// ---- PMIS (amg.cpp:36-86) -----------------------------------------------------
constexpr uint8_t kU = 0, kC = 1, kF = 2;

__global__ void k_indegree(int nnz, const int* __restrict__ col, int* __restrict__ lam) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < nnz) atomicAdd(lam + col[q], 1);
}

__global__ void k_pmis_select(int n, const int* __restrict__ sp, const int* __restrict__ sc,
                              const int* __restrict__ tp, const int* __restrict__ tc,
                              const int* __restrict__ lam, const uint8_t* __restrict__ state,
                              uint8_t* __restrict__ win) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (state[i] != kU) {
    win[i] = 0;
    return;
  }
  const int li = lam[i];
  bool ok = true;
  for (int k = sp[i]; k < sp[i + 1] && ok; ++k) {
    const int j = sc[k];
    if (j == i || state[j] != kU) continue;
    const int lj = lam[j];
    if (!(li > lj || (li == lj && i < j))) ok = false;
  }
  for (int k = tp[i]; k < tp[i + 1] && ok; ++k) {
    const int j = tc[k];
    if (j == i || state[j] != kU) continue;
    const int lj = lam[j];
    if (!(li > lj || (li == lj && i < j))) ok = false;
  }
  win[i] = ok ? 1 : 0;
}

__global__ void k_pmis_mark_c(int n, const uint8_t* __restrict__ win, uint8_t* __restrict__ state,
                              int* __restrict__ nwin) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !win[i]) return;
  state[i] = kC;
  atomicAdd(nwin, 1);
}

__global__ void k_pmis_mark_f(int n, const int* __restrict__ sp, const int* __restrict__ sc,
                              const int* __restrict__ tp, const int* __restrict__ tc,
                              const uint8_t* __restrict__ win, uint8_t* state) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !win[i]) return;
  for (int k = sp[i]; k < sp[i + 1]; ++k)
    if (state[sc[k]] == kU) state[sc[k]] = kF;
  for (int k = tp[i]; k < tp[i + 1]; ++k)
    if (state[tc[k]] == kU) state[tc[k]] = kF;
}

__global__ void k_count_undecided(int n, const uint8_t* __restrict__ state, int* __restrict__ cnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  int u = (i < n && state[i] == kU) ? 1 : 0;
  u = __reduce_add_sync(0xffffffffu, u);
  if ((threadIdx.x & 31) == 0 && u) atomicAdd(cnt, u);
}

__global__ void k_is_c(int n, const uint8_t* __restrict__ state, uint8_t* __restrict__ is_c) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) is_c[i] = state[i] == kC ? 1 : 0;
}

// ---- ranks ---------------------------------------------------------------------
__global__ void k_flag_to_int(int n, const uint8_t* __restrict__ f, int* __restrict__ o) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) o[i] = f[i] ? 1 : 0;
}
__global__ void k_rank(int n, const uint8_t* __restrict__ f, const int* __restrict__ pre,
                       int* __restrict__ cid) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) cid[i] = f[i] ? pre[i] : -1;
}

// ---- direct interpolation (amg.cpp:88-141) --------------------------------------
struct RowStats {
  double aii, rsum, csum, rmax;
};

// Walks A(i,:) in column order with a merge pointer into the (sorted) strength
// row, accumulating exactly as the reference loop does.
__device__ RowStats interp_stats(int i, const int* ptr, const int* col, const double* val,
                                 const int* sp, const int* sc, const int* cid) {
  RowStats r{0.0, 0.0, 0.0, 0.0};
  int sk = sp[i];
  const int se = sp[i + 1];
  for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
    const int j = col[k];
    const double v = val[k];
    r.rmax = stdmax(r.rmax, fabs(v));
    if (j == i) {
      r.aii = v;
      continue;
    }
    r.rsum = __dadd_rn(r.rsum, v);
    while (sk < se && sc[sk] < j) ++sk;
    const bool strong = sk < se && sc[sk] == j;
    if (cid[j] >= 0 && strong) r.csum = __dadd_rn(r.csum, v);
  }
  return r;
}

template <bool kFill>
__global__ void k_interp(int n, const int* __restrict__ ptr, const int* __restrict__ col,
                         const double* __restrict__ val, const int* __restrict__ sp,
                         const int* __restrict__ sc, const int* __restrict__ cid,
                         int* __restrict__ cnt, const int* __restrict__ optr, int* __restrict__ ocol,
                         double* __restrict__ oval, unsigned long long* __restrict__ fallback,
                         int* __restrict__ zero_diag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (cid[i] >= 0) {
    if (kFill) {
      ocol[optr[i]] = cid[i];
      oval[optr[i]] = 1.0;
    } else {
      cnt[i] = 1;
    }
    return;
  }
  const RowStats st = interp_stats(i, ptr, col, val, sp, sc, cid);
  if (st.aii == 0.0) {
    *zero_diag = 1;
    if (!kFill) cnt[i] = 0;
    return;
  }
  const bool usable = fabs(st.csum) > __dmul_rn(1e-14, st.rmax);
  const double scale = usable ? __ddiv_rn(st.rsum, __dmul_rn(st.aii, st.csum)) : 0.0;
  int c = 0;
  int o = kFill ? optr[i] : 0;
  int sk = sp[i];
  const int se = sp[i + 1];
  for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
    const int j = col[k];
    if (j == i || cid[j] < 0) continue;
    while (sk < se && sc[sk] < j) ++sk;
    const bool strong = sk < se && sc[sk] == j;
    if (usable && !strong) continue;
    if (kFill) {
      ocol[o] = cid[j];
      oval[o] = usable ? __dmul_rn(-val[k], scale) : __ddiv_rn(-val[k], st.aii);
      ++o;
    }
    ++c;
  }
  if (!kFill) {
    cnt[i] = c;
    if (!usable) atomicAdd(fallback, 1ull);
  }
}

}  // namespace

DCsr strength_graph(const DCsr& A, double theta, cudaStream_t s) {
  if (A.rows != A.cols) throw InvalidArgument("strength_graph: matrix must be square");
  DCsr S;
  S.rows = S.cols = A.rows;
  S.ptr.alloc(A.rows + 1, s);
  DVec<int> cnt(A.rows > 0 ? A.rows : 1, s);
  if (A.rows) {
    k_strength<false><<<blocks_for(A.rows, 256), 256, 0, s>>>(A.rows, theta, A.ptr.get(), A.col.get(),
                                                             A.val.get(), cnt.get(), nullptr, nullptr,
                                                             nullptr);
    MGRX_LAUNCH_CK();
    count_launch();
  }
  S.nnz = static_cast<int>(exclusive_scan(cnt.get(), S.ptr.get(), A.rows, s));
  S.col.alloc(S.nnz, s);
  S.val.alloc(S.nnz, s);
  if (A.rows) {
    k_strength<true><<<blocks_for(A.rows, 256), 256, 0, s>>>(A.rows, theta, A.ptr.get(), A.col.get(),
                                                            A.val.get(), nullptr, S.ptr.get(),
                                                            S.col.get(), S.val.get());
    MGRX_LAUNCH_CK();
    count_launch();
  }
  return S;
}

int pmis(const DCsr& S, DVec<uint8_t>& is_c, cudaStream_t s) {
  const int n = S.rows;
  is_c.alloc(n, s);
  if (n == 0) return 0;
  DVec<int> lam(n, s);
  lam.zero();
  if (S.nnz) {
    k_indegree<<<blocks_for(S.nnz, 256), 256, 0, s>>>(S.nnz, S.col.get(), lam.get());
    MGRX_LAUNCH_CK();
    count_launch();
  }
  const DCsr St = transpose(S, s);
  DVec<uint8_t> state(n, s), win(n, s);
  state.zero();
  DVec<int> counters(2, s);
  int rounds = 0;
  const int nb = blocks_for(n, 256);
  while (true) {
    counters.zero();
    k_pmis_select<<<nb, 256, 0, s>>>(n, S.ptr.get(), S.col.get(), St.ptr.get(), St.col.get(),
                                     lam.get(), state.get(), win.get());
    k_pmis_mark_c<<<nb, 256, 0, s>>>(n, win.get(), state.get(), counters.get());
    k_pmis_mark_f<<<nb, 256, 0, s>>>(n, S.ptr.get(), S.col.get(), St.ptr.get(), St.col.get(),
                                     win.get(), state.get());
    k_count_undecided<<<nb, 256, 0, s>>>(n, state.get(), counters.get() + 1);
    MGRX_LAUNCH_CK();
    count_launch(4);
    ++rounds;
    const std::vector<int> c = counters.download(2);
    if (c[0] == 0 && c[1] > 0) throw RuntimeError("pmis_coarsen: stalled selection round");
    if (c[1] == 0) break;
  }
  k_is_c<<<nb, 256, 0, s>>>(n, state.get(), is_c.get());
  MGRX_LAUNCH_CK();
  count_launch();
  return rounds;
}

int rank_flags(const uint8_t* flag, int n, DVec<int>& cid, cudaStream_t s) {
  cid.alloc(n > 0 ? n : 1, s);
  if (n == 0) return 0;
  DVec<int> f(n, s), pre(n + 1, s);
  k_flag_to_int<<<blocks_for(n, 256), 256, 0, s>>>(n, flag, f.get());
  MGRX_LAUNCH_CK();
  count_launch();
  const int total = static_cast<int>(exclusive_scan(f.get(), pre.get(), n, s));
  k_rank<<<blocks_for(n, 256), 256, 0, s>>>(n, flag, pre.get(), cid.get());
  MGRX_LAUNCH_CK();
  count_launch();
  return total;
}

DCsr classical_interp(const DCsr& A, const DCsr& S, const int* cid, int nc, long long* fallback,
                      cudaStream_t s) {
  const int n = A.rows;
  DCsr P;
  P.rows = n;
  P.cols = nc;
  P.ptr.alloc(n + 1, s);
  DVec<int> cnt(n > 0 ? n : 1, s), zd(1, s);
  DVec<unsigned long long> fb(1, s);
  zd.zero();
  fb.zero();
  if (n) {
    k_interp<false><<<blocks_for(n, 256), 256, 0, s>>>(n, A.ptr.get(), A.col.get(), A.val.get(),
                                                      S.ptr.get(), S.col.get(), cid, cnt.get(),
                                                      nullptr, nullptr, nullptr, fb.get(), zd.get());
    MGRX_LAUNCH_CK();
    count_launch();
  }
  if (read_scalar(zd.get(), s)) throw RuntimeError("classical_interp: zero diagonal at an F-row");
  P.nnz = static_cast<int>(exclusive_scan(cnt.get(), P.ptr.get(), n, s));
  P.col.alloc(P.nnz, s);
  P.val.alloc(P.nnz, s);
  if (n) {
    k_interp<true><<<blocks_for(n, 256), 256, 0, s>>>(n, A.ptr.get(), A.col.get(), A.val.get(),
                                                     S.ptr.get(), S.col.get(), cid, nullptr,
                                                     P.ptr.get(), P.col.get(), P.val.get(), nullptr,
                                                     zd.get());
    MGRX_LAUNCH_CK();
    count_launch();
  }
  if (fallback) *fallback += static_cast<long long>(read_scalar(fb.get(), s));
  return P;
}

}  // namespace mgrx
