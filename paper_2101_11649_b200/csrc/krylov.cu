// Device GMRES. Each modified Gram-Schmidt step is one fused kernel: it
// applies the previous projection (w -= h_{i-1} v_{i-1}, with h read from HBM
// so nothing waits on the host) and reduces the next inner product v_i . w in
// the same pass. Reductions use a fixed grid and a fixed tree, with the last
// CTA folding the per-CTA partials in index order, so every run is bitwise
// reproducible. The host reads the Hessenberg column once per step (one
// small D2H copy), exactly where the reference needs scalar control flow.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>

#include "krylov.cuh"
#include "relax.cuh"

namespace mgrx {
namespace {

constexpr int kRT = 256;     // threads per reduction CTA
constexpr int kRB = 592;     // reduction CTAs (4 per SM on 148 SMs)

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, o));
  return v;
}

// Fixed-order block reduction of two values; result valid in thread 0.
__device__ void block_sum2(double& a, double& b) {
  __shared__ double sa[kRT / 32], sb[kRT / 32];
  a = warp_sum(a);
  b = warp_sum(b);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    sa[w] = a;
    sb[w] = b;
  }
  __syncthreads();
  if (w == 0) {
    a = l < kRT / 32 ? sa[l] : 0.0;
    b = l < kRT / 32 ? sb[l] : 0.0;
    a = warp_sum(a);
    b = warp_sum(b);
  }
  __syncthreads();
}

// L2 eviction-priority hints (createpolicy + ld/st .L2::cache_hint). The
// Arnoldi vector w (n doubles, 34 MB at cfg2) is read and rewritten by every
// MGS launch of a step; pinning it with evict_last keeps it in the 126 MB L2
// so each launch's HBM traffic is the basis vectors it streams.
__device__ __forceinline__ unsigned long long pol_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long pol_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double ld_pol(const double* a, unsigned long long p) {
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(p));
  return v;
}
__device__ __forceinline__ void st_pol(double* a, double v, unsigned long long p) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(p) : "memory");
}

// kHint: 0 plain (.cg); 1 w evict_last; 2 + vprev evict_first; 3 + a evict_last
// (3 is the default: 7% faster solves at cfg2 than 0).
// w <- w - (*hprev) * vprev (if vprev); then dot1 = sum a_i w_i (if a),
// dot2 = sum w_i w_i (if want2). Results: out1 (and hacc = / += dot1), out2.
template <int kHint>
__global__ void __launch_bounds__(kRT)
    k_mgs(int n, double* __restrict__ w, const double* __restrict__ vprev,
          const double* __restrict__ hprev, const double* __restrict__ a, int want2,
          double* __restrict__ part, unsigned* __restrict__ ctr, double* __restrict__ out1,
          double* __restrict__ hacc, int accumulate, double* __restrict__ out2) {
  const double h = vprev ? *hprev : 0.0;
  double s1 = 0.0, s2 = 0.0;
  // Grid-stride slice of this lane, processed kU iterations at a time: all
  // loads of the group are issued first (memory-level parallelism), then the
  // lane's partial sums are updated in the same sequential order as a plain
  // loop (the canonical reduction order shared with the oracle).
  constexpr int kU = 4;
  constexpr int kStride = kRB * kRT;
  unsigned long long pl = 0, pf = 0;
  if (kHint) {
    pl = pol_last();
    pf = pol_first();
  }
  int i0 = blockIdx.x * kRT + threadIdx.x;
  for (; i0 + (kU - 1) * kStride < n; i0 += kU * kStride) {
    double wv[kU], pv[kU], av[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = i0 + u * kStride;
      wv[u] = kHint >= 1 ? ld_pol(w + i, pl) : __ldcg(w + i);
      if (vprev) pv[u] = kHint >= 2 ? ld_pol(vprev + i, pf) : __ldcg(vprev + i);
      if (a) av[u] = kHint >= 3 ? ld_pol(a + i, pl) : __ldcg(a + i);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      double wi = wv[u];
      if (vprev) {
        wi = __dsub_rn(wi, __dmul_rn(h, pv[u]));
        if (kHint >= 1) st_pol(w + i0 + u * kStride, wi, pl);
        else w[i0 + u * kStride] = wi;
      }
      if (a) s1 = __dadd_rn(s1, __dmul_rn(av[u], wi));
      if (want2) s2 = __dadd_rn(s2, __dmul_rn(wi, wi));
    }
  }
  for (int i = i0; i < n; i += kStride) {
    double wi = w[i];
    if (vprev) {
      wi = __dsub_rn(wi, __dmul_rn(h, vprev[i]));
      w[i] = wi;
    }
    if (a) s1 = __dadd_rn(s1, __dmul_rn(a[i], wi));
    if (want2) s2 = __dadd_rn(s2, __dmul_rn(wi, wi));
  }
  block_sum2(s1, s2);
  __shared__ bool last;
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = s1;
    part[2 * blockIdx.x + 1] = s2;
    __threadfence();
    last = atomicAdd(ctr, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double t1 = 0.0, t2 = 0.0;
  for (int b = threadIdx.x; b < gridDim.x; b += kRT) {
    t1 = __dadd_rn(t1, __ldcg(part + 2 * b));
    t2 = __dadd_rn(t2, __ldcg(part + 2 * b + 1));
  }
  block_sum2(t1, t2);
  if (threadIdx.x == 0) {
    if (a) {
      if (out1) *out1 = t1;
      if (hacc) *hacc = accumulate ? __dadd_rn(*hacc, t1) : t1;
    }
    if (want2 && out2) *out2 = t2;
    *ctr = 0u;
  }
}

__global__ void k_scale(int n, const double* __restrict__ in, double d, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = __ddiv_rn(in[i], d);
}

// u_i = sum_j V[j][i] y_j, j ascending.
__global__ void k_gemv(int n, int k, const double* __restrict__ V, const double* __restrict__ y,
                       double* __restrict__ u) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int j = 0; j < k; ++j) s = __dadd_rn(s, __dmul_rn(V[static_cast<size_t>(j) * n + i], y[j]));
  u[i] = s;
}

void mgs_launch(int n, double* w, const double* vprev, const double* hprev, const double* a,
                bool want2, GmresWork& ws, double* out1, double* hacc, bool accumulate, double* out2,
                cudaStream_t s) {
  static const int hint = [] {
    const char* v = std::getenv("MGRX_MGS_L2");
    return v ? std::atoi(v) : 3;
  }();
  auto* kern = hint == 0 ? k_mgs<0> : hint == 1 ? k_mgs<1> : hint == 2 ? k_mgs<2> : k_mgs<3>;
  kern<<<kRB, kRT, 0, s>>>(n, w, vprev, hprev, a, want2 ? 1 : 0, ws.part.get(), ws.ctr.get(), out1, hacc,
                           accumulate ? 1 : 0, out2);
  MGRX_LAUNCH_CK();
  count_launch();
}

// ---------------------------------------------------------------------------
// Fused Arnoldi step: the whole modified Gram-Schmidt of one GMRES step
// (both passes, the re-orthogonalisation test and the scaling of v_{k+1}) in
// ONE persistent cooperative kernel. w never leaves the SMs: 148 CTAs x 1024
// threads hold it in shared memory (<= 28 doubles per thread, 224 KB per SM),
// so each projection streams only v_i from HBM (plus its L2 re-read for the
// update) and the n-vector round trips of w disappear.
//
// Lane numbering is the canonical reduction order's: thread T of CTA c is
// lane c*1024+T = canonical block 4c+T/256, thread T%256, owning rows
// lane + q*kStride. Per-lane sums, the 256-lane block trees and the in-order
// fold of the 592 block partials are the same floating-point operations
// k_mgs performs, so results are bitwise identical to the launch-per-
// projection path (and to the oracle).
constexpr int kAT = 1024;
constexpr int kAB = kRB * kRT / kAT;  // 148
constexpr int kAMaxSlots = 28;
constexpr int kAU = 4;    // row slots per load group (loads of a group are issued together)
constexpr int kAHk = 64;  // Hessenberg entries the writer keeps in shared memory

struct ArnoldiArgs {
  int n, k;
  double* w;          // in: A M^-1 v_k
  const double* V;    // basis, column-major n x (m+1)
  double* part;       // 2 x kRB x 2 partials (double-buffered by phase)
  unsigned* bar;      // grid barrier counter (zeroed before launch)
  double* n0;         // ||w||^2 before pass 1
  double* n1;         // final ||w||^2
  double* hp;         // per-projection dots of the last pass
  double* hc;         // Hessenberg column H(0..k, k)
  int dbg;            // probe only: 1 skip the row loops, 2 skip the grid barrier, 4 force two passes, 8 trace
  // sharded: cross-rank exchange of each phase's rank partial (nranks > 1)
  int nranks = 1, rank = 0;
  double* mbox = nullptr;             // this rank's mailbox
  double* const* peers = nullptr;     // every rank's mailbox (device array)
  unsigned long long epoch = 0;       // tag base of this launch
  double* err = nullptr;              // set to 1 on a peer timeout
  // lane-pair kernel: merge pass 1's norm phase with pass 2's first
  // projection (one grid reduction fewer per re-orthogonalised step)
  int merge = 0;
  double* npass = nullptr;            // out: passes run (1 or 2)
};

// One projection phase over this lane's rows (w in shared memory, column
// stride kAT): w -= h*vprev (kV); s1 += av.w (kA); s2 += w.w (kW2).
template <bool kV, bool kA, bool kW2>
__device__ __forceinline__ void arn_rows(double* wl, int nslot, const double* __restrict__ pl,
                                         const double* __restrict__ al, double h, unsigned long long pf,
                                         double& s1, double& s2) {
  constexpr int kStride = kRB * kRT;
  int q = 0;
  for (; q + kAU - 1 < nslot; q += kAU) {
    double pv[kAU], xv[kAU];
#pragma unroll
    for (int u = 0; u < kAU; ++u) {
      if (kV) pv[u] = ld_pol(pl + (q + u) * kStride, pf);
      if (kA) xv[u] = __ldcg(al + (q + u) * kStride);
    }
#pragma unroll
    for (int u = 0; u < kAU; ++u) {
      double wi = wl[(q + u) * kAT];
      if (kV) {
        wi = __dsub_rn(wi, __dmul_rn(h, pv[u]));
        wl[(q + u) * kAT] = wi;
      }
      if (kA) s1 = __dadd_rn(s1, __dmul_rn(xv[u], wi));
      if (kW2) s2 = __dadd_rn(s2, __dmul_rn(wi, wi));
    }
  }
  for (; q < nslot; ++q) {
    double wi = wl[q * kAT];
    if (kV) {
      wi = __dsub_rn(wi, __dmul_rn(h, ld_pol(pl + q * kStride, pf)));
      wl[q * kAT] = wi;
    }
    if (kA) s1 = __dadd_rn(s1, __dmul_rn(__ldcg(al + q * kStride), wi));
    if (kW2) s2 = __dadd_rn(s2, __dmul_rn(wi, wi));
  }
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(kAT, 1) k_arnoldi(ArnoldiArgs a) {
  extern __shared__ double wsm[];  // [slot][kAT]
  __shared__ double r1[kAT / 32], r2[kAT / 32];  // per-warp sums of this CTA
  __shared__ double f1[kRT / 32], f2[kRT / 32];  // fold: per-warp sums of the kRB partials
  const int T = threadIdx.x;
  const int wp = T >> 5, l = T & 31;
  const int n = a.n, k = a.k;
  constexpr int kStride = kRB * kRT;
  const int lane = blockIdx.x * kAT + T;
  const int nslot = lane < n ? (n - 1 - lane) / kStride + 1 : 0;
  for (int q = 0; q < nslot; ++q) wsm[q * kAT + T] = __ldcg(a.w + lane + q * kStride);
  const unsigned long long pf = pol_first();
  const size_t ld = static_cast<size_t>(n);
  double* wl = wsm + T;

  unsigned phase = 0;
  // Reduce (s1, s2) over the grid in the canonical order (dbg & 8: CTAs 0 and
  // last print a per-phase globaltimer breakdown).
  const bool tracer = (a.dbg & 8) && T == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1);
  unsigned long long tprev = tracer ? gtimer() : 0, tm[4];
  auto reduce = [&](double s1, double s2, double& t1, double& t2) {
    if (tracer) tm[0] = gtimer();
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if (l == 0) {
      r1[wp] = s1;
      r2[wp] = s2;
    }
    __syncthreads();
    double* part = a.part + (phase & 1) * 2 * kRB;
    if (wp < kAT / kRT) {  // canonical 256-lane block trees (block_sum2)
      double x1 = l < kRT / 32 ? r1[wp * (kRT / 32) + l] : 0.0;
      double x2 = l < kRT / 32 ? r2[wp * (kRT / 32) + l] : 0.0;
      x1 = warp_sum(x1);
      x2 = warp_sum(x2);
      if (l == 0) {
        const int b = blockIdx.x * (kAT / kRT) + wp;
        part[2 * b] = x1;
        part[2 * b + 1] = x2;
      }
    }
    __syncthreads();
    if (tracer) tm[1] = gtimer();
    // grid barrier (monotonic counter; zeroed by the host before the launch)
    if (T == 0 && !(a.dbg & 2)) {
      __threadfence();
      atomicAdd(a.bar, 1u);
      const unsigned target = (phase + 1) * gridDim.x;
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.bar) : "memory");
      } while (v < target);
    }
    __syncthreads();
    if (tracer) tm[2] = gtimer();
    // every CTA folds the kRB partials in index order (k_mgs's last block);
    // all loads of a thread are issued before the in-order adds
    if (T < kRT) {
      constexpr int kF = (kRB + kRT - 1) / kRT;
      double p1[kF], p2[kF];
#pragma unroll
      for (int j = 0; j < kF; ++j) {
        const int b = T + j * kRT;
        if (b < kRB) {
          p1[j] = __ldcg(part + 2 * b);
          p2[j] = __ldcg(part + 2 * b + 1);
        }
      }
      double u1 = 0.0, u2 = 0.0;
#pragma unroll
      for (int j = 0; j < kF; ++j) {
        if (T + j * kRT < kRB) {
          u1 = __dadd_rn(u1, p1[j]);
          u2 = __dadd_rn(u2, p2[j]);
        }
      }
      u1 = warp_sum(u1);
      u2 = warp_sum(u2);
      if (l == 0) {
        f1[wp] = u1;
        f2[wp] = u2;
      }
    }
    __syncthreads();
    // every warp completes the fold itself; lane 0 holds the canonical value
    const double x1 = l < kRT / 32 ? f1[l] : 0.0;
    const double x2 = l < kRT / 32 ? f2[l] : 0.0;
    t1 = __shfl_sync(0xffffffffu, warp_sum(x1), 0);
    t2 = __shfl_sync(0xffffffffu, warp_sum(x2), 0);
    if (tracer) {
      tm[3] = gtimer();
      printf("ARN cta %d phase %u loop %llu part %llu bar %llu fold %llu\n", blockIdx.x, phase, tm[0] - tprev,
             tm[1] - tm[0], tm[2] - tm[1], tm[3] - tm[2]);
      tprev = gtimer();
    }
    ++phase;
  };

  const bool writer = blockIdx.x == 0 && T == 0;
  __shared__ double hk[kAHk];  // writer: H(i,k) of pass 1 (i < kAHk)
  double h = 0.0, wn2 = 0.0, w02 = 0.0;
  for (int pass = 0; pass < 2; ++pass) {
    for (int i = 0; i <= k + 1; ++i) {  // i == k + 1: the closing norm
      double s1 = 0.0, s2 = 0.0, t1, t2;
      if (!(a.dbg & 1)) {
        const double* pl = i ? a.V + (i - 1) * ld + lane : nullptr;
        const double* al = a.V + i * ld + lane;
        if (i > k) arn_rows<true, false, true>(wl, nslot, pl, al, h, pf, s1, s2);
        else if (i) arn_rows<true, true, false>(wl, nslot, pl, al, h, pf, s1, s2);
        else if (pass == 0) arn_rows<false, true, true>(wl, nslot, pl, al, h, pf, s1, s2);
        else arn_rows<false, true, false>(wl, nslot, pl, al, h, pf, s1, s2);
      }
      reduce(s1, s2, t1, t2);
      if (i <= k) {
        if (pass == 0 && i == 0) w02 = t2;
        h = t1;
        if (writer) {
          a.hp[i] = t1;
          const double hv = pass ? __dadd_rn(i < kAHk ? hk[i] : a.hc[i], t1) : t1;
          if (i < kAHk) hk[i] = hv;
          a.hc[i] = hv;
        }
      } else {
        wn2 = t2;
      }
    }
    h = 0.0;
    // re-orthogonalise when ||w|| drops below ||w0|| / sqrt(2) (krylov.cpp:90)
    if (pass == 1 || (!(a.dbg & 4) && !(__dsqrt_rn(wn2) < __ddiv_rn(__dsqrt_rn(w02), __dsqrt_rn(2.0))))) break;
  }
  if (writer) {
    *a.n0 = w02;
    *a.n1 = wn2;
  }
  const double wn = __dsqrt_rn(wn2);
  if (!(wn < 1e-300)) {
    double* out = const_cast<double*>(a.V) + (k + 1) * ld;
    for (int q = 0; q < nslot; ++q) out[lane + q * kStride] = __ddiv_rn(wsm[q * kAT + T], wn);
  }
}

// ---------------------------------------------------------------------------
// Lane-pair variant (the default): 512 threads per CTA, thread t of CTA c
// owns canonical lanes c*1024 + 2t and 2t+1, so every access is a 16-byte
// pair and each thread has 128 registers. The row loop of a projection is
// bound by memory-level parallelism, not by HBM bandwidth: the 1024-thread
// kernel (64 registers) keeps 4 slots x 16 B per thread in flight, ~32 KB of
// HBM reads per SM, which covers ~0.6 of the HBM latency-bandwidth product.
// Here a group of kU slots issues kU x 32 B per thread (HBM v_i + L2 v_{i-1})
// before any is consumed.
//
// The canonical reduction is reproduced exactly: per lane, the products are
// summed in slot order into separate accumulators (x: lane 2t, y: lane
// 2t+1); the canonical warp tree (shfl_down 16, 8, 4, 2, 1 over 32 lanes)
// maps onto a 16-thread half warp as shfl_down 8, 4, 2, 1 applied to x and y
// separately followed by x + y (canonical lane 0 + lane 1); the 256-lane
// block trees and the fold of the 592 block partials are unchanged.
constexpr int kAT2 = 512;

__device__ __forceinline__ double2 ld2_pol(const double* a, unsigned long long p) {
  double2 v;
  asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(a), "l"(p));
  return v;
}

// Canonical 32-lane warp sum of the lanes held by one 16-thread half warp
// (valid in threads 0 and 16 of the warp).
__device__ __forceinline__ double half_warp_pair_sum(double x, double y) {
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) {
    x = __dadd_rn(x, __shfl_down_sync(0xffffffffu, x, o));
    y = __dadd_rn(y, __shfl_down_sync(0xffffffffu, y, o));
  }
  return __dadd_rn(x, y);
}

struct PairSums {
  double s1x = 0.0, s1y = 0.0, s2x = 0.0, s2y = 0.0;
};

template <bool kV, bool kA, bool kW2>
__device__ __forceinline__ void arn2_slot(double2* wp, double2 pv, double2 xv, double h, PairSums& s) {
  double2 wi = *wp;
  if (kV) {
    wi.x = __dsub_rn(wi.x, __dmul_rn(h, pv.x));
    wi.y = __dsub_rn(wi.y, __dmul_rn(h, pv.y));
    *wp = wi;
  }
  if (kA) {
    s.s1x = __dadd_rn(s.s1x, __dmul_rn(xv.x, wi.x));
    s.s1y = __dadd_rn(s.s1y, __dmul_rn(xv.y, wi.y));
  }
  if (kW2) {
    s.s2x = __dadd_rn(s.s2x, __dmul_rn(wi.x, wi.x));
    s.s2y = __dadd_rn(s.s2y, __dmul_rn(wi.y, wi.y));
  }
}

// One projection phase over this thread's lane pair: nsy slots where both
// lanes hold a row, plus (xtail) one more slot for lane x only.
template <int kU, bool kV, bool kA, bool kW2>
__device__ __forceinline__ void arn2_rows(double2* wl, int nsy, bool xtail, const double* __restrict__ pl,
                                          const double* __restrict__ al, double h, unsigned long long pf,
                                          PairSums& s, int rot = 0) {
  constexpr int kStride = kRB * kRT;
  int q = 0;
  for (; q + kU <= nsy; q += kU) {
    double2 pv[kU], xv[kU];
    int qs[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      qs[u] = q + u + rot;  // rot != 0: timing experiment only (slot order rotated per CTA)
      if (qs[u] >= nsy) qs[u] -= nsy;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (kV) pv[u] = pl ? ld2_pol(pl + qs[u] * kStride, pf) : make_double2(0.0, 0.0);
      if (kA) xv[u] = __ldcg(reinterpret_cast<const double2*>(al + qs[u] * kStride));
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) arn2_slot<kV, kA, kW2>(wl + qs[u] * kAT2, pv[u], xv[u], h, s);
  }
  for (; q < nsy; ++q) {
    double2 pv = make_double2(0.0, 0.0), xv = make_double2(0.0, 0.0);
    if (kV && pl) pv = ld2_pol(pl + q * kStride, pf);
    if (kA) xv = __ldcg(reinterpret_cast<const double2*>(al + q * kStride));
    arn2_slot<kV, kA, kW2>(wl + q * kAT2, pv, xv, h, s);
  }
  if (xtail) {
    double* wx = reinterpret_cast<double*>(wl + q * kAT2);
    double wi = *wx;
    if (kV) {
      wi = __dsub_rn(wi, __dmul_rn(h, __ldcg(pl + q * kStride)));
      *wx = wi;
    }
    if (kA) s.s1x = __dadd_rn(s.s1x, __dmul_rn(__ldcg(al + q * kStride), wi));
    if (kW2) s.s2x = __dadd_rn(s.s2x, __dmul_rn(wi, wi));
  }
}

__device__ __forceinline__ unsigned long long gtime_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Sharded: publish this rank's partial of the phase into every rank's
// mailbox slot [phase][rank] (CTA 0; data, then the tag with release), wait
// for every rank's tag in the local mailbox, and fold the partials in rank
// order as k_fold2 does (v = p_0; v += p_q for q = 1..). Every CTA folds the
// same values, so all CTAs and all ranks hold the same bits.
__device__ __noinline__ void cross_rank(const ArnoldiArgs& a, unsigned phase, double& t1, double& t2) {
  __shared__ double m1[kMboxRanks], m2[kMboxRanks];  // this phase's rank partials
  const int T = threadIdx.x;
  const int slot = static_cast<int>(phase % kMboxPhases);
  // once this rank has flagged a timeout it publishes the poison tag, so a
  // peer that is still waiting flags the step too (no rank folds stale values)
  const bool poisoned = *reinterpret_cast<volatile double*>(a.err) != 0.0;
  const unsigned long long tag = poisoned ? kMboxPoison : a.epoch + phase + 1;
  if (blockIdx.x == 0 && T < a.nranks) {
    double* dst = a.peers[T] + (static_cast<size_t>(slot) * kMboxRanks + a.rank) * 4;
    dst[0] = t1;
    dst[1] = t2;
    // release: the two values are visible to the peer before the tag
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(dst + 2), "l"(tag) : "memory");
  }
  if (T < a.nranks) {
    const double* src = a.mbox + (static_cast<size_t>(slot) * kMboxRanks + T) * 4;
    unsigned long long v;
    const unsigned long long t0 = gtime_ns();
    bool late = false;
    for (unsigned it = 0;; ++it) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(src + 2) : "memory");
      if (v == tag && !poisoned) break;
      if (v == kMboxPoison) {
        late = true;
        break;
      }
      // a silent peer: give up after ~2 s (or at once when a previous phase
      // already did) and flag the step; the host discards it
      if ((it & 1023u) == 1023u &&
          (gtime_ns() - t0 > 2000000000ull || *reinterpret_cast<volatile double*>(a.err) != 0.0)) {
        late = true;
        break;
      }
    }
    double p1, p2;
    asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(p1) : "l"(src) : "memory");
    asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(p2) : "l"(src + 1) : "memory");
    m1[T] = p1;
    m2[T] = p2;
    if (late) {
      *a.err = 1.0;
      // poison this phase's slot of every peer as well (CTA 0 only)
      if (blockIdx.x == 0) {
        double* dst = a.peers[T] + (static_cast<size_t>(slot) * kMboxRanks + a.rank) * 4;
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(dst + 2), "l"(kMboxPoison) : "memory");
      }
    }
  }
  __syncthreads();
  double v1 = m1[0], v2 = m2[0];
  for (int q = 1; q < a.nranks; ++q) {
    v1 = __dadd_rn(v1, m1[q]);
    v2 = __dadd_rn(v2, m2[q]);
  }
  t1 = v1;
  t2 = v2;
  // m1/m2 are next written after the next phase's block barriers
}

// Grid-wide reduction of one projection phase in the canonical order (see
// above): canonical warp sums, 256-lane block trees, partials, grid barrier,
// in-order fold of the kRB partials in every CTA. r/f: shared scratch.
template <bool kShard>
__device__ __forceinline__ void pair_reduce(const ArnoldiArgs& a, const PairSums& ps, unsigned phase, double* r1,
                                            double* r2, double* f1, double* f2, double& t1, double& t2) {
  const int T = threadIdx.x;
  const int wp = T >> 5, l = T & 31;
  const double c1 = half_warp_pair_sum(ps.s1x, ps.s1y);
  const double c2 = half_warp_pair_sum(ps.s2x, ps.s2y);
  if ((T & 15) == 0) {  // canonical warp T/16 of this CTA
    r1[T >> 4] = c1;
    r2[T >> 4] = c2;
  }
  __syncthreads();
  double* part = a.part + (phase & 1) * 2 * kRB;
  if (wp < kAT / kRT) {  // canonical 256-lane block trees (block_sum2)
    double x1 = l < kRT / 32 ? r1[wp * (kRT / 32) + l] : 0.0;
    double x2 = l < kRT / 32 ? r2[wp * (kRT / 32) + l] : 0.0;
    x1 = warp_sum(x1);
    x2 = warp_sum(x2);
    if (l == 0) {
      const int b = blockIdx.x * (kAT / kRT) + wp;
      part[2 * b] = x1;
      part[2 * b + 1] = x2;
    }
  }
  __syncthreads();
  if (T == 0 && !(a.dbg & 2)) {
    __threadfence();
    atomicAdd(a.bar, 1u);
    const unsigned target = (phase + 1) * gridDim.x;
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.bar) : "memory");
    } while (v < target);
  }
  __syncthreads();
  if (T < kRT) {
    constexpr int kF = (kRB + kRT - 1) / kRT;
    double p1[kF], p2[kF];
#pragma unroll
    for (int j = 0; j < kF; ++j) {
      const int b = T + j * kRT;
      if (b < kRB) {
        p1[j] = __ldcg(part + 2 * b);
        p2[j] = __ldcg(part + 2 * b + 1);
      }
    }
    double u1 = 0.0, u2 = 0.0;
#pragma unroll
    for (int j = 0; j < kF; ++j) {
      if (T + j * kRT < kRB) {
        u1 = __dadd_rn(u1, p1[j]);
        u2 = __dadd_rn(u2, p2[j]);
      }
    }
    u1 = warp_sum(u1);
    u2 = warp_sum(u2);
    if (l == 0) {
      f1[wp] = u1;
      f2[wp] = u2;
    }
  }
  __syncthreads();
  const double x1 = l < kRT / 32 ? f1[l] : 0.0;
  const double x2 = l < kRT / 32 ? f2[l] : 0.0;
  t1 = __shfl_sync(0xffffffffu, warp_sum(x1), 0);
  t2 = __shfl_sync(0xffffffffu, warp_sum(x2), 0);
  if (kShard) cross_rank(a, phase, t1, t2);
}

// Writer bookkeeping of one reduced phase (H column, norms).
__device__ __forceinline__ void arn_record(const ArnoldiArgs& a, bool writer, int pass, int i, double t1, double t2,
                                           double* hk, double& h, double& w02, double& wn2) {
  if (i <= a.k) {
    if (pass == 0 && i == 0) w02 = t2;
    h = t1;
    if (writer) {
      a.hp[i] = t1;
      const double hv = pass ? __dadd_rn(i < kAHk ? hk[i] : a.hc[i], t1) : t1;
      if (i < kAHk) hk[i] = hv;
      a.hc[i] = hv;
    }
  } else {
    wn2 = t2;
  }
}

template <int kU, bool kShard = false>
__global__ void __launch_bounds__(kAT2, 1) k_arnoldi2(ArnoldiArgs a) {
  extern __shared__ double2 wsm2[];               // [slot][kAT2] lane pairs
  __shared__ double r1[kAT / 32], r2[kAT / 32];   // canonical warp sums of this CTA (32)
  __shared__ double f1[kRT / 32], f2[kRT / 32];   // fold: per-warp sums of the kRB partials
  __shared__ double hk[kAHk];
  const int T = threadIdx.x;
  const int n = a.n, k = a.k;
  constexpr int kStride = kRB * kRT;
  const int lane = blockIdx.x * kAT + 2 * T;  // lane x; lane y = lane + 1 (n is even: both or neither)
  const int nsy = lane < n ? (n - 1 - lane) / kStride + 1 : 0;
  for (int q = 0; q < nsy; ++q)
    wsm2[q * kAT2 + T] = __ldcg(reinterpret_cast<const double2*>(a.w + lane + q * kStride));
  const unsigned long long pf = pol_first();
  const size_t ld = static_cast<size_t>(n);
  double2* wl = wsm2 + T;
  const bool writer = blockIdx.x == 0 && T == 0;
  double h = 0.0, wn2 = 0.0, w02 = 0.0;
  unsigned phase = 0;
  // Merged phase (a.merge, set by the host when the previous step needed the
  // second pass): pass 1's last phase (w -= h_k v_k; ||w||^2) also forms
  // v_0 . w, which is exactly pass 2's first projection (same w, same slot
  // order, same reduction: bitwise). If the test then skips pass 2, that dot
  // is discarded (one extra column read).
  const bool merge = !kShard && a.merge;
  double h0 = 0.0;
  int passes = 1;
  for (int pass = 0; pass < 2; ++pass) {
    for (int i = (pass == 1 && merge) ? 1 : 0; i <= k + 1; ++i) {
      const bool mphase = merge && pass == 0 && i == k + 1;
      PairSums ps;
      double t1, t2;
      if (!(a.dbg & 1)) {
        // dbg & 64 (timing experiment, not bitwise): no L2 re-read of v_{i-1}
        const double* pl = (i && !(a.dbg & 64)) ? a.V + (i - 1) * ld + lane : nullptr;
        const double* al = a.V + (mphase ? 0 : i) * ld + lane;
        // dbg & 32 (timing experiment, not bitwise): rotate the slot order per CTA
        const int rot = (a.dbg & 32) ? (kU * (blockIdx.x % (nsy / kU > 0 ? nsy / kU : 1))) % (nsy > 0 ? nsy : 1) : 0;
        if (mphase) arn2_rows<kU, true, true, true>(wl, nsy, false, pl, al, h, pf, ps, rot);
        else if (i > k) arn2_rows<kU, true, false, true>(wl, nsy, false, pl, al, h, pf, ps, rot);
        else if (i) arn2_rows<kU, true, true, false>(wl, nsy, false, pl, al, h, pf, ps, rot);
        else if (pass == 0) arn2_rows<kU, false, true, true>(wl, nsy, false, pl, al, h, pf, ps, rot);
        else arn2_rows<kU, false, true, false>(wl, nsy, false, pl, al, h, pf, ps, rot);
      }
      pair_reduce<kShard>(a, ps, phase++, r1, r2, f1, f2, t1, t2);
      if (mphase) {
        wn2 = t2;
        h0 = t1;
      } else {
        arn_record(a, writer, pass, i, t1, t2, hk, h, w02, wn2);
      }
    }
    h = 0.0;
    if (pass == 1 || (!(a.dbg & 4) && !(__dsqrt_rn(wn2) < __ddiv_rn(__dsqrt_rn(w02), __dsqrt_rn(2.0))))) break;
    passes = 2;
    if (merge) arn_record(a, writer, 1, 0, h0, 0.0, hk, h, w02, wn2);  // pass 2, projection 0
  }
  if (writer) {
    *a.n0 = w02;
    *a.n1 = wn2;
    if (a.npass) *a.npass = passes;
  }
  const double wn = __dsqrt_rn(wn2);
  if (!(wn < 1e-300)) {
    double* out = const_cast<double*>(a.V) + (k + 1) * ld;
    for (int q = 0; q < nsy; ++q) {
      const double2 wi = wsm2[q * kAT2 + T];
      reinterpret_cast<double2*>(out + lane + q * kStride)[0] = make_double2(__ddiv_rn(wi.x, wn), __ddiv_rn(wi.y, wn));
    }
  }
}

// MGRX_ARNOLDI: 0 off (launch-per-projection MGS), 1 the 1024-thread kernel,
// 2 (default) the lane-pair kernel with MGRX_ARNOLDI_U slots per load group
// (4, 6 or 8; default 4: 6 and 8 measured 2-5% slower per step at cfg2). The lane-pair kernel needs 16-byte aligned basis
// columns (n even); odd n uses the 1024-thread kernel.
struct ArnoldiMode {
  int mode = 2, u = 4;
  bool fits1 = false, fits2 = false;
};

template <typename K>
bool arnoldi_fits(K kern, int threads) {
  const int bytes = kAMaxSlots * kAT * static_cast<int>(sizeof(double));
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, bytes) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return occ >= 1;
}

// Per device (kernel attributes and SM counts are per device).
const ArnoldiMode& arnoldi_mode() {
  static std::mutex mu;
  static std::map<int, ArnoldiMode> modes;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = modes.find(dev);
  if (it != modes.end()) return it->second;
  ArnoldiMode r;
  if (const char* v = std::getenv("MGRX_ARNOLDI")) r.mode = std::atoi(v);
  if (const char* v = std::getenv("MGRX_ARNOLDI_U")) r.u = std::atoi(v);
  if (r.u != 4 && r.u != 6) r.u = 8;
  if (device_sms() == kAB) {
    r.fits1 = arnoldi_fits(k_arnoldi, kAT);
    r.fits2 = arnoldi_fits(r.u == 4 ? k_arnoldi2<4> : r.u == 6 ? k_arnoldi2<6> : k_arnoldi2<8>, kAT2);
  }
  return modes.emplace(dev, r).first->second;
}

// MGRX_ARNOLDI_MERGE=0: never merge the pass-1 norm phase with pass 2's
// first projection.
bool arnoldi_merge_on() {
  static const bool on = [] {
    const char* v = std::getenv("MGRX_ARNOLDI_MERGE");
    return !v || std::atoi(v) != 0;
  }();
  return on;
}

int arnoldi_slots(int n) {
  const ArnoldiMode& m = arnoldi_mode();
  constexpr int kStride = kRB * kRT;
  if (!m.mode || n <= 0) return 0;
  const bool pair = m.mode >= 2 && m.fits2 && n % 2 == 0;
  if (!pair && !m.fits1) return 0;
  const int slots = (n - 1) / kStride + 1;
  return slots <= kAMaxSlots ? slots : 0;
}

// merge: see k_arnoldi2 (lane-pair kernel only). The pass count lands in
// scalar slot 2m+5, inside the Hessenberg-column D2H.
void arnoldi_launch(int n, int k, int slots, int dbg, GmresWork& ws, cudaStream_t s, bool merge = false) {
  double* S = ws.scal.get();
  const int m = ws.m;
  MGRX_CK(cudaMemsetAsync(ws.bar.get(), 0, sizeof(unsigned), s));
  ArnoldiArgs aa{n, k, ws.w.get(), ws.V.get(), ws.apart.get(), ws.bar.get(), S, S + 1, S + 2, S + 3 + (m + 1), dbg};
  aa.merge = merge && arnoldi_merge_on() ? 1 : 0;
  aa.npass = S + 2 * m + 5;
  void* args[] = {&aa};
  const ArnoldiMode& md = arnoldi_mode();
  const size_t smem = static_cast<size_t>(slots) * kAT * sizeof(double);
  if (md.mode >= 2 && md.fits2 && n % 2 == 0 && !(dbg & 8)) {
    void* kern = md.u == 4 ? reinterpret_cast<void*>(k_arnoldi2<4>)
                 : md.u == 6 ? reinterpret_cast<void*>(k_arnoldi2<6>)
                             : reinterpret_cast<void*>(k_arnoldi2<8>);
    MGRX_CK(cudaLaunchCooperativeKernel(kern, dim3(kAB), dim3(kAT2), args, smem, s));
  } else {
    MGRX_CK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_arnoldi), dim3(kAB), dim3(kAT), args, smem, s));
  }
  count_launch();
}

}  // namespace

bool arnoldi_sharded_ok(int n) {
  const ArnoldiMode& md = arnoldi_mode();
  return md.mode >= 2 && md.fits2 && n > 0 && n % 2 == 0 && arnoldi_slots(n) > 0;
}

void arnoldi_sharded(int n, int k, int dbg, const ArnoldiPeers& pe, GmresWork& ws, cudaStream_t s) {
  if (!arnoldi_sharded_ok(n) || pe.nranks > kMboxRanks) throw RuntimeError("sharded Arnoldi kernel unavailable");
  const int slots = arnoldi_slots(n);
  double* S = ws.scal.get();
  const int m = ws.m;
  MGRX_CK(cudaMemsetAsync(ws.bar.get(), 0, sizeof(unsigned), s));
  MGRX_CK(cudaMemsetAsync(S + m + 3, 0, sizeof(double), s));
  ArnoldiArgs aa{n, k, ws.w.get(), ws.V.get(), ws.apart.get(), ws.bar.get(), S, S + 1, S + 2, S + 3 + (m + 1), dbg};
  aa.nranks = pe.nranks;
  aa.rank = pe.rank;
  aa.mbox = pe.mbox;
  aa.peers = pe.peers;
  aa.epoch = pe.epoch;
  aa.err = S + m + 3;
  void* args[] = {&aa};
  const ArnoldiMode& md = arnoldi_mode();
  if (first_on_device(reinterpret_cast<const void*>(k_arnoldi2<4, true>))) {
    const int bytes = kAMaxSlots * kAT * static_cast<int>(sizeof(double));
    MGRX_CK(cudaFuncSetAttribute(k_arnoldi2<4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  }
  (void)md;
  MGRX_CK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_arnoldi2<4, true>), dim3(kAB), dim3(kAT2), args,
                                      static_cast<size_t>(slots) * kAT * sizeof(double), s));
  count_launch();
}


void mgs_step(int n, double* w, const double* vprev, const double* hprev, const double* a, bool want2,
              GmresWork& ws, double* out1, double* hacc, bool accumulate, double* out2, cudaStream_t s) {
  mgs_launch(n, w, vprev, hprev, a, want2, ws, out1, hacc, accumulate, out2, s);
}

void vec_scale(int n, const double* in, double d, double* out, cudaStream_t s) {
  if (n == 0) return;
  k_scale<<<blocks_for(n, 256), 256, 0, s>>>(n, in, d, out);
  MGRX_LAUNCH_CK();
  count_launch();
}

void basis_combine(int n, int k, const double* V, const double* y, double* u, cudaStream_t s) {
  if (n == 0) return;
  k_gemv<<<blocks_for(n, 256), 256, 0, s>>>(n, k, V, y, u);
  MGRX_LAUNCH_CK();
  count_launch();
}

void GmresWork::ensure(int n_, int m_, cudaStream_t s) {
  if (n_ == n && m_ == m) return;
  n = n_;
  m = m_;
  V.alloc(static_cast<size_t>(n) * (m + 1), s);
  w.alloc(n, s);
  r.alloc(n, s);
  z.alloc(n, s);
  u.alloc(n, s);
  scal.alloc(4 + 3 * (m + 2), s);
  scal.zero();
  part.alloc(2 * kRB, s);
  ctr.alloc(1, s);
  ctr.zero();
  apart.alloc(4 * kRB, s);
  bar.alloc(1, s);

  if (hpinned) cudaFreeHost(hpinned);
  MGRX_CK(cudaMallocHost(&hpinned, sizeof(double) * (4 + 3 * (m + 2))));
}

GmresWork::~GmresWork() {
  if (hpinned) cudaFreeHost(hpinned);
}

void mgs_probe(int n, double* w, const double* vprev, const double* h, const double* a, GmresWork& ws,
               cudaStream_t s) {
  mgs_launch(n, w, vprev, h, a, false, ws, ws.scal.get() + 2, nullptr, false, nullptr, s);
}

int arnoldi_probe(int n, int k, int dbg, GmresWork& ws, cudaStream_t s) {
  const int slots = arnoldi_slots(n);
  if (!slots || k < 0 || k >= ws.m) return 0;
  arnoldi_launch(n, k, slots, dbg, ws, s, true);
  return 1;
}

double device_dot(int n, const double* a, const double* b, GmresWork& ws, cudaStream_t s) {
  // dot(a, b) = sum a_i b_i via the MGS kernel with w = b, no projection.
  mgs_launch(n, const_cast<double*>(b), nullptr, nullptr, a, false, ws, ws.scal.get(), nullptr,
             false, nullptr, s);
  return read_scalar(ws.scal.get(), s);
}

namespace {
// MGRX_GMRES_PROF=1: per-step event timeline of the fused-Arnoldi loop,
// printed at the end of the solve (prec / spmv / arnoldi / D2H / gap from the
// previous step's D2H to this step's first kernel = host bubble).
struct StepProf {
  bool on = false;
  cudaEvent_t ev[5] = {};
  cudaEvent_t last = nullptr;
  double acc[5] = {};
  int steps = 0;
  StepProf() {
    const char* v = std::getenv("MGRX_GMRES_PROF");
    on = v && v[0] == '1';
    if (!on) return;
    for (auto& e : ev) cudaEventCreate(&e);
    cudaEventCreate(&last);
  }
  void rec(int i, cudaStream_t s) { cudaEventRecord(ev[i], s); }
  void step() {
    float t[5] = {};
    if (steps > 0) cudaEventElapsedTime(&t[0], last, ev[0]);
    for (int i = 1; i < 5; ++i) cudaEventElapsedTime(&t[i], ev[i - 1], ev[i]);
    for (int i = 0; i < 5; ++i) acc[i] += t[i];
    std::swap(last, ev[4]);
    ++steps;
  }
  ~StepProf() {
    if (!on) return;
    std::fprintf(stderr, "GMRES_PROF steps %d ms: gap %.3f prec %.3f spmv %.3f arnoldi %.3f d2h %.3f\n", steps, acc[0],
                 acc[1], acc[2], acc[3], acc[4]);
    for (auto& e : ev) cudaEventDestroy(e);
    cudaEventDestroy(last);
  }
};
}  // namespace

bool self_exchange() {
  static const bool on = [] {
    const char* v = std::getenv("MGRX_ARNOLDI_SELFXCHG");
    return v && v[0] == '1';
  }();
  return on;
}

GmresResult gmres_device(const DCsr& A, const double* b, double* x, const KrylovSpec& cfg,
                         const DevOp& precond, GmresWork& ws, cudaStream_t s, const DevOp& precond_capture) {
  const int n = A.rows;
  if (cfg.restart < 1) throw InvalidArgument("gmres: restart must be >= 1");
  if (cfg.ortho != kOrthoMgs && lowsync_supported(n, cfg.restart))
    return gmres_lowsync(A, b, x, cfg, precond, precond_capture, ws, s);
  NvtxRange nvtx("mgrx.gmres.mgs");
  StepProf prof;
  const int m = cfg.restart;
  ws.ensure(n, m, s);
  double* S = ws.scal.get();
  // scalar slots: [0] norm^2 a, [1] norm^2 b, [2, 2+m+1) pass h, [3+m+1 ...) H column
  double* s_n0 = S;
  double* s_n1 = S + 1;
  double* s_hp = S + 2;
  double* s_hc = S + 3 + (m + 1);
  double* H_pin = ws.hpinned;
  const size_t col_bytes = sizeof(double) * (3 + 2 * (m + 1) + 1);

  GmresResult res;
  auto prec = [&](const double* in, double* out) {
    if (precond) precond(in, out, s);
    else MGRX_CK(cudaMemcpyAsync(out, in, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  };
  auto norm2 = [&](const double* v) {
    mgs_launch(n, const_cast<double*>(v), nullptr, nullptr, nullptr, true, ws, nullptr, nullptr, false,
               s_n0, s);
    return read_scalar(s_n0, s);
  };

  {
    // rhs finiteness + norm (krylov.cpp:42-51)
    const double bb = norm2(b);
    if (!std::isfinite(bb)) throw RuntimeError("gmres: rhs contains non-finite entries");
    const double bnorm = std::sqrt(bb);
    if (bnorm == 0.0) {
      MGRX_CK(cudaMemsetAsync(x, 0, sizeof(double) * n, s));
      res.converged = true;
      return res;
    }
    const double target = std::max(cfg.rel_tol * bnorm, cfg.abs_tol);
    std::vector<double> H(static_cast<size_t>(m + 1) * m, 0.0), cs(m, 0.0), sn(m, 0.0), g(m + 1, 0.0);
    auto h = [&](int i, int j) -> double& { return H[static_cast<size_t>(j) * (m + 1) + i]; };
    double* V = ws.V.get();
    auto col = [&](int j) { return V + static_cast<size_t>(j) * n; };

    bool merge_next = true;  // the previous step ran the second MGS pass
    while (res.iterations < cfg.max_iters) {
      spmv_residual(A, x, b, nullptr, ws.r.get(), s);  // r = b - A x
      const double rnorm = std::sqrt(norm2(ws.r.get()));
      if (!std::isfinite(rnorm)) throw RuntimeError("gmres: residual is non-finite");
      if (rnorm <= target) {
        res.converged = true;
        res.final_residual = rnorm / bnorm;
        res.history.push_back(res.final_residual);
        return res;
      }
      k_scale<<<blocks_for(n, 256), 256, 0, s>>>(n, ws.r.get(), rnorm, col(0));
      MGRX_LAUNCH_CK();
      count_launch();
      std::fill(g.begin(), g.end(), 0.0);
      g[0] = rnorm;
      int k = 0;
      bool breakdown = false;
      for (; k < m && res.iterations < cfg.max_iters; ++k) {
        if (prof.on) prof.rec(0, s);
        prec(col(k), ws.z.get());
        if (prof.on) prof.rec(1, s);
        spmv(A, ws.z.get(), ws.w.get(), s);  // w = A M^{-1} v_k
        if (prof.on) prof.rec(2, s);
        double wn;
        if (const int slots = arnoldi_slots(n)) {
          // both MGS passes + re-orthogonalisation test + v_{k+1} in one kernel
          if (self_exchange() && arnoldi_sharded_ok(n)) {
            // test mode (MGRX_ARNOLDI_SELFXCHG=1): the sharded kernel as a
            // one-rank group exchanging with its own mailbox
            static double* mbox = nullptr;
            static double** peers = nullptr;
            static unsigned long long epoch = 0;
            if (!mbox) {
              MGRX_CK(cudaMalloc(&mbox, sizeof(double) * kMboxDoubles));
              MGRX_CK(cudaMemset(mbox, 0, sizeof(double) * kMboxDoubles));
              MGRX_CK(cudaMalloc(&peers, sizeof(double*)));
              MGRX_CK(cudaMemcpy(peers, &mbox, sizeof(double*), cudaMemcpyHostToDevice));
            }
            ArnoldiPeers pe;
            pe.nranks = 1;
            pe.mbox = mbox;
            pe.peers = peers;
            epoch += 1ull << 16;
            pe.epoch = epoch;
            arnoldi_sharded(n, k, 0, pe, ws, s);
          } else {
            arnoldi_launch(n, k, slots, 0, ws, s, merge_next);
          }
          if (prof.on) prof.rec(3, s);
          MGRX_CK(cudaMemcpyAsync(H_pin, S, col_bytes, cudaMemcpyDeviceToHost, s));
          if (prof.on) prof.rec(4, s);
          MGRX_CK(cudaStreamSynchronize(s));
          if (prof.on) prof.step();
          if (self_exchange() && H_pin[m + 3] != 0.0) throw RuntimeError("Arnoldi self-exchange timed out");
          wn = std::sqrt(H_pin[1]);
          merge_next = H_pin[2 * m + 5] == 2.0;
        } else {
          // pass 1: h_i = v_i . w ; w -= h_i v_i  (krylov.cpp:84-89)
          for (int i = 0; i <= k; ++i)
            mgs_launch(n, ws.w.get(), i ? col(i - 1) : nullptr, i ? s_hp + (i - 1) : nullptr, col(i),
                       i == 0, ws, s_hp + i, s_hc + i, false, i == 0 ? s_n0 : nullptr, s);
          mgs_launch(n, ws.w.get(), col(k), s_hp + k, nullptr, true, ws, nullptr, nullptr, false, s_n1, s);
          MGRX_CK(cudaMemcpyAsync(H_pin, S, col_bytes, cudaMemcpyDeviceToHost, s));
          MGRX_CK(cudaStreamSynchronize(s));
          const double w0 = std::sqrt(H_pin[0]);
          wn = std::sqrt(H_pin[1]);
          if (wn < w0 / std::sqrt(2.0)) {
            // pass 2 (krylov.cpp:90-96): H(i,k) += h_i
            for (int i = 0; i <= k; ++i)
              mgs_launch(n, ws.w.get(), i ? col(i - 1) : nullptr, i ? s_hp + (i - 1) : nullptr, col(i),
                         false, ws, s_hp + i, s_hc + i, true, nullptr, s);
            mgs_launch(n, ws.w.get(), col(k), s_hp + k, nullptr, true, ws, nullptr, nullptr, false, s_n1, s);
            MGRX_CK(cudaMemcpyAsync(H_pin, S, col_bytes, cudaMemcpyDeviceToHost, s));
            MGRX_CK(cudaStreamSynchronize(s));
            wn = std::sqrt(H_pin[1]);
          }
          if (!(wn < 1e-300)) {
            k_scale<<<blocks_for(n, 256), 256, 0, s>>>(n, ws.w.get(), wn, col(k + 1));
            MGRX_LAUNCH_CK();
            count_launch();
          }
        }
        const double* hc = H_pin + 3 + (m + 1);
        for (int i = 0; i <= k; ++i) h(i, k) = hc[i];
        h(k + 1, k) = wn;
        if (!std::isfinite(wn)) throw RuntimeError("gmres: Arnoldi vector is non-finite");
        const bool happy = wn < 1e-300;
        // Givens (krylov.cpp:11-33)
        for (int i = 0; i < k; ++i) {
          const double t = cs[i] * h(i, k) + sn[i] * h(i + 1, k);
          h(i + 1, k) = -sn[i] * h(i, k) + cs[i] * h(i + 1, k);
          h(i, k) = t;
        }
        const double aa = h(k, k), bb2 = h(k + 1, k);
        const double rr = std::hypot(aa, bb2);
        if (rr == 0.0) {
          cs[k] = 1.0;
          sn[k] = 0.0;
        } else {
          cs[k] = aa / rr;
          sn[k] = bb2 / rr;
        }
        h(k, k) = rr;
        h(k + 1, k) = 0.0;
        const double t = cs[k] * g[k];
        g[k + 1] = -sn[k] * g[k];
        g[k] = t;
        ++res.iterations;
        const double est = std::abs(g[k + 1]);
        res.history.push_back(est / bnorm);
        if (happy) {
          breakdown = true;
          ++k;
          break;
        }
        if (est <= target) {
          ++k;
          break;
        }
      }
      int keff = k;
      while (keff > 0 && std::abs(h(keff - 1, keff - 1)) < 1e-300) --keff;
      if (keff > 0) {
        std::vector<double> y(keff);
        for (int i = keff - 1; i >= 0; --i) {
          double acc = g[i];
          for (int j = i + 1; j < keff; ++j) acc -= h(i, j) * y[j];
          y[i] = acc / h(i, i);
        }
        MGRX_CK(cudaMemcpyAsync(s_hp, y.data(), sizeof(double) * keff, cudaMemcpyHostToDevice, s));
        k_gemv<<<blocks_for(n, 256), 256, 0, s>>>(n, keff, V, s_hp, ws.u.get());
        MGRX_LAUNCH_CK();
        count_launch();
        prec(ws.u.get(), ws.z.get());
        vec_add(n, ws.z.get(), x, s);  // x += M^{-1}(V y)
        MGRX_CK(cudaStreamSynchronize(s));  // y lives on the host stack
      }
      spmv_residual(A, x, b, nullptr, ws.r.get(), s);
      const double tn = std::sqrt(norm2(ws.r.get()));
      if (!std::isfinite(tn)) throw RuntimeError("gmres: residual is non-finite");
      res.history.push_back(tn / bnorm);
      if (tn <= target) {
        res.converged = true;
        res.final_residual = tn / bnorm;
        return res;
      }
      if (breakdown) throw RuntimeError("gmres: Arnoldi breakdown before reaching tolerance");
      res.final_residual = tn / bnorm;
    }
  }
  return res;
}

}  // namespace mgrx
