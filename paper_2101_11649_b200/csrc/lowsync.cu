// Low-synchronisation orthogonalisation for the device GMRES (ortho "cgs2",
// the default; the reference's modified Gram-Schmidt stays available as
// ortho "mgs", bitwise against the oracle).
//
// The reference step (proj/src/krylov.cpp:80-101) projects w = A M^-1 v_k
// onto v_0..v_k one vector at a time (MGS), then once more when ||w|| fell
// below ||w0||/sqrt(2). On the GPU every projection is a grid-wide
// reduction: 2k+4 dependent reductions per step, each streaming one basis
// column, so the step is bound by synchronisation (0.43 of HBM at cfg2).
//
// Here a step is TWO sweeps over the basis and one grid reduction each
// (lagged classical Gram-Schmidt with re-orthogonalisation, "DCGS2"):
//
//   step k holds U = w'_{k-1}, the once-orthogonalised, UNnormalised next
//   vector of step k-1, and w = A M^-1 U (the preconditioner and the SpMV
//   ran on U).
//   sweep A (k_ls_dots):   s = V_{k-1}^T U, t = V_{k-1}^T w, alpha = U.w,
//                          nu = U.U                    (one reduction)
//       gamma = sqrt(nu - s.s)      v_k = (U - V_{k-1} s) / gamma
//       (U = gamma v_k + V_{k-1} s finalises column k-1 of H:
//        H(0..k-1, k-1) += s, H(k, k-1) = gamma)
//       A M^-1 v_k = (w - V_k Hbar_{k-1} s) / gamma, so
//       h = V_k^T A M^-1 v_k = ([t; (alpha - s.t)/gamma] - Hbar s) / gamma
//   sweep B (k_ls_update): v_k = (U - V_{k-1} s)/gamma  -> basis column k
//                          w' = w/gamma - V_{k-1} t/gamma - v_k (alpha - s.t)/gamma^2
//                             = (I - V_k V_k^T) A M^-1 v_k  -> U
//                          beta^2 = w'.w'              (one reduction)
//
// i.e. the re-orthogonalisation of v_k rides on the next step's sweeps
// (always two passes, which the reference's 1/sqrt(2) test runs whenever
// it triggers). Column k of H is preliminary (h, beta) until step k+1
// finalises it; the Givens rotation of the preliminary column gives the
// residual estimate of step k (the reference's convergence test,
// krylov.cpp:103-117) and is recomputed from the final column one step
// later. Every scalar of this bookkeeping (H, the rotations, g, the
// history, the stopping flags) lives on the device: the host reads nothing
// per step, and a whole restart cycle runs as one CUDA graph with a
// conditional WHILE node (MGRX_GMRES_GRAPH=0: host-driven loop, one
// 64-byte read per step).
//
// Bytes per step: 16 n (k+3) (sweep A reads V_{k-1}, U, w; sweep B reads
// them again and writes v_k and U), with U and w held in L2 between the
// sweeps (evict_last). No grid barrier, no cooperative launch, no limit on
// n or on the SM count, odd n allowed (the basis has a padded leading
// dimension). Reductions use a fixed partition and fixed trees:
// deterministic run to run on a given GPU model.
//
// Parity: not bitwise with the reference's MGS (different, equally stable
// orthogonalisation); the north_star bar (history within 1e-10 for the first
// 10 steps, iterations +-1, final true residual <= rtol) is asserted against
// the oracle in tests/test_gpu_fullsize.py and tests/test_gpu_parity.py.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "krylov.cuh"
#include "relax.cuh"

namespace mgrx {

struct LsArgs {
  int n, ldv, m, G;
  int G2;             // sweep B grid (2 CTAs per SM)
  double* V;          // basis, column-major, leading dimension ldv
  double* U;          // next vector (in: U_k, out: U_{k+1})
  const double* w;    // A M^-1 U_k
  double* part;       // sweep A partials [(2m+2) values][G]
  double* part2;      // sweep B partials [G]
  unsigned* ticket;   // [0] sweep A, [1] sweep B (last-CTA election)
  LsState* st;
  double* Hraw;       // (m+1) x m, column-major: final columns < k, preliminary column k
  double* Hrot;       // rotated H (tentative rotation on the last column)
  double* cs;
  double* sn;
  double* g;          // rotated rhs, final through index k
  double* coef;       // sweep A -> B: s[0..k), d[0..k] at m.., 1/gamma at 2m+1
  double* hist;       // per-cycle residual estimates (relative)
  double* rank_part;  // sharded: this rank's folded partials (null: single GPU, fused finish)
  cudaGraphConditionalHandle cond;
  int use_cond;
};

namespace {
constexpr int kLT = 256;  // threads per CTA
constexpr int kLW = kLT / 32;
constexpr int kLC = 8;    // basis columns per register chunk (16 spills)



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
__device__ __forceinline__ double2 ld2(const double* a, unsigned long long p) {
  double2 v;
  asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(a), "l"(p));
  return v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// This CTA's row pairs [pb, pe) (a fixed partition of the n/2 pairs); the
// odd last row (n odd) belongs to the last CTA.
__device__ __forceinline__ void cta_pairs(const LsArgs& a, long long& pb, long long& pe, int G) {
  const long long np = a.n / 2;
  pb = np * blockIdx.x / G;
  pe = np * (blockIdx.x + 1) / G;
}

// Sweep A over basis columns [c0, c0 + nc) (nc <= NC; NC == 0: alpha and nu
// only). RU row pairs per thread per iteration keep 16-20 loads in flight.
// Columns beyond the first chunk re-read U and w, from L2 (evict_last).
// Per-thread sums in a fixed order, warp xor trees, warps in index order.
// Exactly NC columns (no predicates: the loads of a group of RU row pairs
// are all issued before the first use).
template <int NC, int RU, bool kFirst>
__device__ __forceinline__ void dots_group(const LsArgs& a, const double* Vc, long long p, double* s, double* t,
                                           double& al, double& nu, unsigned long long pl, unsigned long long pf) {
  double2 uv[RU], wv[RU], vv[RU][NC > 0 ? NC : 1];
#pragma unroll
  for (int r = 0; r < RU; ++r) {
    const long long pr = p + static_cast<long long>(r) * kLT;
    uv[r] = ld2(a.U + 2 * pr, pl);
    wv[r] = ld2(a.w + 2 * pr, pl);
#pragma unroll
    for (int j = 0; j < NC; ++j) vv[r][j] = ld2(Vc + static_cast<size_t>(j) * a.ldv + 2 * pr, pf);
  }
#pragma unroll
  for (int r = 0; r < RU; ++r) {
    if (kFirst) {
      al = fma(uv[r].x, wv[r].x, al);
      al = fma(uv[r].y, wv[r].y, al);
      nu = fma(uv[r].x, uv[r].x, nu);
      nu = fma(uv[r].y, uv[r].y, nu);
    }
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      s[j] = fma(vv[r][j].x, uv[r].x, s[j]);
      s[j] = fma(vv[r][j].y, uv[r].y, s[j]);
      t[j] = fma(vv[r][j].x, wv[r].x, t[j]);
      t[j] = fma(vv[r][j].y, wv[r].y, t[j]);
    }
  }
}

template <int NC, int RU, bool kFirst>
__device__ __forceinline__ void dots_chunk(const LsArgs& a, int k, int c0, double* red) {
  long long pb, pe;
  cta_pairs(a, pb, pe, a.G);
  const unsigned long long pl = pol_last(), pf = pol_first();
  double s[NC > 0 ? NC : 1], t[NC > 0 ? NC : 1], al = 0.0, nu = 0.0;
#pragma unroll
  for (int j = 0; j < NC; ++j) s[j] = t[j] = 0.0;
  const double* Vc = a.V + static_cast<size_t>(c0) * a.ldv;
  long long p = pb + threadIdx.x;
  // full groups of RU row pairs, then the remaining pairs one at a time
  for (; p + static_cast<long long>(RU - 1) * kLT < pe; p += static_cast<long long>(kLT) * RU)
    dots_group<NC, RU, kFirst>(a, Vc, p, s, t, al, nu, pl, pf);
  for (; p < pe; p += kLT) dots_group<NC, 1, kFirst>(a, Vc, p, s, t, al, nu, pl, pf);
  if ((a.n & 1) && blockIdx.x == a.G - 1 && threadIdx.x == 0) {  // odd last row
    const int i = a.n - 1;
    const double u = a.U[i], wv = a.w[i];
    if (kFirst) {
      al = fma(u, wv, al);
      nu = fma(u, u, nu);
    }
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      const double v = Vc[static_cast<size_t>(j) * a.ldv + i];
      s[j] = fma(v, u, s[j]);
      t[j] = fma(v, wv, t[j]);
    }
  }
  // block reduction: red[warp][value], values 2j (s_j), 2j+1 (t_j), 2NC (alpha), 2NC+1 (nu)
  constexpr int NV = 2 * NC + 2;
  const int wp = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    const double x = warp_sum(s[j]), y = warp_sum(t[j]);
    if (l == 0) {
      red[wp * NV + 2 * j] = x;
      red[wp * NV + 2 * j + 1] = y;
    }
  }
  if (kFirst) {
    const double x = warp_sum(al), y = warp_sum(nu);
    if (l == 0) {
      red[wp * NV + 2 * NC] = x;
      red[wp * NV + 2 * NC + 1] = y;
    }
  }
  __syncthreads();
  const int T = threadIdx.x;
  if (T < (kFirst ? NV : 2 * NC)) {
    double v = red[T];
    for (int q = 1; q < kLW; ++q) v += red[q * NV + T];
    // global value index: s_j -> 2(c0+j), t_j -> 2(c0+j)+1, alpha -> 2k, nu -> 2k+1
    const int gi = T < 2 * NC ? 2 * c0 + T : 2 * k + (T - 2 * NC);
    a.part[static_cast<size_t>(gi) * a.G + blockIdx.x] = v;
  }
  __syncthreads();
}

__device__ __forceinline__ double& HR(const LsArgs& a, int i, int j) { return a.Hraw[static_cast<size_t>(j) * (a.m + 1) + i]; }
__device__ __forceinline__ double& HT(const LsArgs& a, int i, int j) { return a.Hrot[static_cast<size_t>(j) * (a.m + 1) + i]; }

// Last CTA of sweep A: fold the per-CTA partials of value v in CTA index
// order into tot[v] (shared memory).
__device__ void fold_cta_partials(const LsArgs& a, int nv, double* tot) {
  for (int v = threadIdx.x; v < nv; v += kLT) {
    const double* p = a.part + static_cast<size_t>(v) * a.G;
    double acc = 0.0;
    int c = 0;
    for (; c + 8 <= a.G; c += 8) {
      double x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = __ldcg(p + c + u);
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += x[u];
    }
    for (; c < a.G; ++c) acc += __ldcg(p + c);
    tot[v] = acc;
  }
  __syncthreads();
}

// From the reduced dots tot[] (s_i at 2i, t_i at 2i+1, alpha at 2k, nu at
// 2k+1): finalise column k-1, form the preliminary column k and the sweep-B
// coefficients (one CTA). q: shared scratch of m+1.
__device__ void coef_math(const LsArgs& a, int k, const double* tot, double* q) {
  __shared__ double sh_g, sh_e;
  if (threadIdx.x == 0) {
    double ss = 0.0, st = 0.0;
    for (int i = 0; i < k; ++i) {
      ss = fma(tot[2 * i], tot[2 * i], ss);
      st = fma(tot[2 * i], tot[2 * i + 1], st);
    }
    const double al = tot[2 * k], nu = tot[2 * k + 1];
    const double g2 = nu - ss;
    double gam = g2 > 0.0 ? sqrt(g2) : 0.0;
    if (!(gam > 0.0) || !isfinite(gam)) {
      a.st->flags |= kLsNonFinite | kLsCycleEnd;
      gam = 1.0;  // keep the arithmetic finite; the host throws
    }
    sh_g = gam;
    sh_e = (al - st) / gam;  // v_k . w
    a.st->gamma = gam;
    if (k == 0) a.g[0] = gam;
    else HR(a, k, k - 1) = gam;
  }
  __syncthreads();
  const double gam = sh_g;
  for (int i = threadIdx.x; i < k; i += kLT) HR(a, i, k - 1) += tot[2 * i];  // finalise column k-1
  __syncthreads();
  for (int i = threadIdx.x; i <= k; i += kLT) {  // q = Hbar_{k-1} s
    double acc = 0.0;
    for (int j = i > 0 ? i - 1 : 0; j < k; ++j) acc = fma(HR(a, i, j), tot[2 * j], acc);
    q[i] = acc;
  }
  __syncthreads();
  for (int i = threadIdx.x; i <= k; i += kLT) {
    const double ti = i < k ? tot[2 * i + 1] : sh_e;
    HR(a, i, k) = (ti - q[i]) / gam;  // preliminary column k
    if (i < k) a.coef[i] = tot[2 * i];
    a.coef[a.m + i] = ti / gam;
  }
  if (threadIdx.x == 0) a.coef[2 * a.m + 1] = 1.0 / gam;
}

__device__ void dots_finish(const LsArgs& a, int k) {
  extern __shared__ double sm[];  // [2m+2] totals, [m+1] q
  double* tot = sm;
  fold_cta_partials(a, 2 * k + 2, tot);
  if (a.rank_part) {  // sharded: publish this rank's sums; k_ls_coef finishes
    for (int v = threadIdx.x; v < 2 * k + 2; v += kLT) a.rank_part[v] = tot[v];
    return;
  }
  coef_math(a, k, tot, sm + 2 * a.m + 2);
}

// Chunk of nc (1..kLC) columns: one exact instantiation per count; RU keeps
// 14-24 loads of 16 B in flight per thread.
template <bool kFirst>
__device__ __forceinline__ void dots_pass(const LsArgs& a, int k, int c0, int nc, double* red) {
  switch (nc) {
    case 1: dots_chunk<1, 6, kFirst>(a, k, c0, red); break;
    case 2: dots_chunk<2, 4, kFirst>(a, k, c0, red); break;
    case 3: dots_chunk<3, 4, kFirst>(a, k, c0, red); break;
    case 4: dots_chunk<4, 3, kFirst>(a, k, c0, red); break;
    case 5: dots_chunk<5, 2, kFirst>(a, k, c0, red); break;
    case 6: dots_chunk<6, 2, kFirst>(a, k, c0, red); break;
    case 7: dots_chunk<7, 2, kFirst>(a, k, c0, red); break;
    default: dots_chunk<8, 2, kFirst>(a, k, c0, red); break;
  }
}

__global__ void __launch_bounds__(kLT, 1) k_ls_dots(LsArgs a) {
  pdl_enter();
  __shared__ double red[kLW * (2 * kLC + 2)];
  const int k = a.st->k;
  if (k == 0) {
    dots_chunk<0, 8, true>(a, 0, 0, red);
  } else {
    for (int c0 = 0; c0 < k; c0 += kLC) {
      const int nc = k - c0 < kLC ? k - c0 : kLC;
      if (c0 == 0) dots_pass<true>(a, k, c0, nc, red);
      else dots_pass<false>(a, k, c0, nc, red);
    }
  }
  __shared__ bool last;
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(&a.ticket[0], 1u) == static_cast<unsigned>(a.G) - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  dots_finish(a, k);
  if (threadIdx.x == 0) a.ticket[0] = 0u;
}

// Givens bookkeeping of step k (one thread): final rotation of column k-1,
// tentative rotation of the preliminary column k, residual estimate,
// stopping flags (krylov.cpp:11-33, 103-117).
__device__ void step_finish(const LsArgs& a, int k, double beta) {
  LsState* st = a.st;
  if (k >= 1) {
    const int j = k - 1;
    for (int i = 0; i <= j + 1; ++i) HT(a, i, j) = HR(a, i, j);
    for (int i = 0; i < j; ++i) {
      const double t = a.cs[i] * HT(a, i, j) + a.sn[i] * HT(a, i + 1, j);
      HT(a, i + 1, j) = -a.sn[i] * HT(a, i, j) + a.cs[i] * HT(a, i + 1, j);
      HT(a, i, j) = t;
    }
    const double aa = HT(a, j, j), bb = HT(a, j + 1, j);
    const double rr = hypot(aa, bb);
    a.cs[j] = rr == 0.0 ? 1.0 : aa / rr;
    a.sn[j] = rr == 0.0 ? 0.0 : bb / rr;
    HT(a, j, j) = rr;
    HT(a, j + 1, j) = 0.0;
    const double t = a.cs[j] * a.g[j];
    a.g[j + 1] = -a.sn[j] * a.g[j];
    a.g[j] = t;
  }
  for (int i = 0; i <= k; ++i) HT(a, i, k) = HR(a, i, k);
  HT(a, k + 1, k) = beta;
  for (int i = 0; i < k; ++i) {
    const double t = a.cs[i] * HT(a, i, k) + a.sn[i] * HT(a, i + 1, k);
    HT(a, i + 1, k) = -a.sn[i] * HT(a, i, k) + a.cs[i] * HT(a, i + 1, k);
    HT(a, i, k) = t;
  }
  const double aa = HT(a, k, k);
  const double rr = hypot(aa, beta);
  const double c = rr == 0.0 ? 1.0 : aa / rr, s = rr == 0.0 ? 0.0 : beta / rr;
  HT(a, k, k) = rr;
  HT(a, k + 1, k) = 0.0;
  st->gt0 = c * a.g[k];
  st->gt1 = -s * a.g[k];
  const double est = fabs(st->gt1);
  st->beta = beta;
  a.hist[st->steps] = est / st->bnorm;
  st->steps += 1;
  st->k = k + 1;
  int f = st->flags;
  if (!isfinite(beta) || !isfinite(est)) f |= kLsNonFinite;
  else if (beta < 1e-300) f |= kLsHappy;
  else if (est <= st->target) f |= kLsConverged;
  if ((f & (kLsNonFinite | kLsHappy | kLsConverged)) || st->k == a.m || st->steps >= st->iters_left) f |= kLsCycleEnd;
  st->flags = f;
  if (a.use_cond) cudaGraphSetConditional(a.cond, (f & kLsCycleEnd) ? 0u : 1u);
}

// Sweep B: exactly NJ basis columns from j0 for RU row pairs (all loads of
// the group issued before use).
template <int NJ, int RU>
__device__ __forceinline__ void upd_group(const LsArgs& a, const double* s, const double* d, int j0, long long p,
                                          double2* av, double2* aw, unsigned long long pf) {
  double2 vv[RU][NJ];
#pragma unroll
  for (int r = 0; r < RU; ++r)
#pragma unroll
    for (int jj = 0; jj < NJ; ++jj)
      vv[r][jj] = ld2(a.V + static_cast<size_t>(j0 + jj) * a.ldv + 2 * (p + static_cast<long long>(r) * kLT), pf);
#pragma unroll
  for (int jj = 0; jj < NJ; ++jj) {
    const double sj = s[j0 + jj], dj = d[j0 + jj];
#pragma unroll
    for (int r = 0; r < RU; ++r) {
      av[r].x = fma(-sj, vv[r][jj].x, av[r].x);
      av[r].y = fma(-sj, vv[r][jj].y, av[r].y);
      aw[r].x = fma(-dj, vv[r][jj].x, aw[r].x);
      aw[r].y = fma(-dj, vv[r][jj].y, aw[r].y);
    }
  }
}

// RU row pairs from p: v_k = (U - V s) / gamma -> column k,
// w' = w / gamma - V d - d_k v_k -> U, acc2 += w'.w'.
template <int RU>
__device__ __forceinline__ void upd_rows(const LsArgs& a, int k, const double* cf, long long p, double& acc2,
                                         unsigned long long pf) {
  const double ig = cf[2 * a.m + 1], dk = cf[a.m + k];
  const double* s = cf;
  const double* d = cf + a.m;
  double2 av[RU], aw[RU];
#pragma unroll
  for (int r = 0; r < RU; ++r) {
    const long long pr = p + static_cast<long long>(r) * kLT;
    av[r] = ld2(a.U + 2 * pr, pf);
    aw[r] = ld2(a.w + 2 * pr, pf);
  }
#pragma unroll
  for (int r = 0; r < RU; ++r) {
    aw[r].x *= ig;
    aw[r].y *= ig;
  }
  int j0 = 0;
  for (; j0 + 8 <= k; j0 += 8) upd_group<8, RU>(a, s, d, j0, p, av, aw, pf);
  switch (k - j0) {
    case 1: upd_group<1, RU>(a, s, d, j0, p, av, aw, pf); break;
    case 2: upd_group<2, RU>(a, s, d, j0, p, av, aw, pf); break;
    case 3: upd_group<3, RU>(a, s, d, j0, p, av, aw, pf); break;
    case 4: upd_group<4, RU>(a, s, d, j0, p, av, aw, pf); break;
    case 5: upd_group<5, RU>(a, s, d, j0, p, av, aw, pf); break;
    case 6: upd_group<6, RU>(a, s, d, j0, p, av, aw, pf); break;
    case 7: upd_group<7, RU>(a, s, d, j0, p, av, aw, pf); break;
    default: break;
  }
  double* Vk = a.V + static_cast<size_t>(k) * a.ldv;
#pragma unroll
  for (int r = 0; r < RU; ++r) {
    const long long pr = p + static_cast<long long>(r) * kLT;
    const double2 vk = make_double2(av[r].x * ig, av[r].y * ig);
    const double2 wp = make_double2(fma(-dk, vk.x, aw[r].x), fma(-dk, vk.y, aw[r].y));
    reinterpret_cast<double2*>(Vk)[pr] = vk;
    reinterpret_cast<double2*>(a.U)[pr] = wp;
    acc2 = fma(wp.x, wp.x, acc2);
    acc2 = fma(wp.y, wp.y, acc2);
  }
}

template <int RU>
__device__ __forceinline__ void update_rows(const LsArgs& a, int k, const double* cf, double& acc2) {
  long long pb, pe;
  cta_pairs(a, pb, pe, a.G2);
  const unsigned long long pf = pol_first();
  long long p = pb + threadIdx.x;
  for (; p + static_cast<long long>(RU - 1) * kLT < pe; p += static_cast<long long>(kLT) * RU)
    upd_rows<RU>(a, k, cf, p, acc2, pf);
  for (; p < pe; p += kLT) upd_rows<1>(a, k, cf, p, acc2, pf);
  if ((a.n & 1) && blockIdx.x == a.G2 - 1 && threadIdx.x == 0) {  // odd last row
    const double ig = cf[2 * a.m + 1], dk = cf[a.m + k];
    const int i = a.n - 1;
    double v = a.U[i], ww = a.w[i] * ig;
    for (int j = 0; j < k; ++j) {
      const double x = a.V[static_cast<size_t>(j) * a.ldv + i];
      v = fma(-cf[j], x, v);
      ww = fma(-cf[a.m + j], x, ww);
    }
    v *= ig;
    ww = fma(-dk, v, ww);
    a.V[static_cast<size_t>(k) * a.ldv + i] = v;
    a.U[i] = ww;
    acc2 = fma(ww, ww, acc2);
  }
}

__global__ void __launch_bounds__(kLT, 2) k_ls_update(LsArgs a) {
  pdl_enter();
  extern __shared__ double cf[];  // coef copy: 2m+2
  const int k = a.st->k;
  for (int i = threadIdx.x; i < 2 * a.m + 2; i += kLT) cf[i] = __ldcg(a.coef + i);
  __syncthreads();
  double acc2 = 0.0;
  if (k <= 4) update_rows<4>(a, k, cf, acc2);
  else update_rows<2>(a, k, cf, acc2);
  __shared__ double red[kLW];
  const double x = warp_sum(acc2);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) {
    double v = red[0];
    for (int q = 1; q < kLW; ++q) v += red[q];
    a.part2[blockIdx.x] = v;
    __threadfence();
    last = atomicAdd(&a.ticket[1], 1u) == static_cast<unsigned>(a.G2) - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x == 0) {
    double b2 = 0.0;
    for (int c = 0; c < a.G2; ++c) b2 += __ldcg(a.part2 + c);
    if (a.rank_part) a.rank_part[0] = b2;  // sharded: k_ls_finish completes the step
    else step_finish(a, k, sqrt(b2));
    a.ticket[1] = 0u;
  }
}

// Sharded: the ranks' sums (gathered[q * stride + v]) folded in rank order,
// then the coefficient math (one CTA; every rank computes the same bits).
__global__ void __launch_bounds__(kLT, 1) k_ls_coef(LsArgs a, const double* __restrict__ gathered, int nranks,
                                                   int stride) {
  pdl_enter();
  extern __shared__ double sm[];
  double* tot = sm;
  const int k = a.st->k;
  for (int v = threadIdx.x; v < 2 * k + 2; v += kLT) {
    double acc = gathered[v];
    for (int q = 1; q < nranks; ++q) acc += gathered[static_cast<size_t>(q) * stride + v];
    tot[v] = acc;
  }
  __syncthreads();
  coef_math(a, k, tot, sm + 2 * a.m + 2);
}

__global__ void k_ls_finish(LsArgs a, const double* __restrict__ gathered, int nranks, int stride) {
  pdl_enter();
  double b2 = gathered[0];
  for (int q = 1; q < nranks; ++q) b2 += gathered[static_cast<size_t>(q) * stride];
  step_finish(a, a.st->k, sqrt(b2));
}

// x-update combination u = V(:, 0..k) y (ld = ldv), j ascending.
__global__ void k_ls_combine(int n, int ldv, int k, const double* __restrict__ V, const double* __restrict__ y,
                             double* __restrict__ u) {
  pdl_enter();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int j = 0; j < k; ++j) s = fma(V[static_cast<size_t>(j) * ldv + i], y[j], s);
  u[i] = s;
}

LsArgs make_args(LsWork& L, int n, int m, double* w) {
  LsArgs a{};
  a.n = n;
  a.ldv = L.ldv;
  a.m = m;
  a.G = L.G;
  a.G2 = 2 * L.G;
  a.V = L.V.get();
  a.U = L.U.get();
  a.w = w;
  a.part = L.part.get();
  a.part2 = L.part2.get();
  a.ticket = L.ticket.get();
  a.st = L.st.get();
  double* D = L.dbl.get();
  a.Hraw = D;
  a.Hrot = D + (m + 1) * m;
  a.cs = D + 2 * (m + 1) * m;
  a.sn = a.cs + m;
  a.g = a.sn + m;
  a.coef = a.g + m + 1;
  a.hist = a.coef + 2 * m + 2;
  return a;
}

size_t dots_smem(int m) { return sizeof(double) * (3 * m + 3); }
size_t update_smem(int m) { return sizeof(double) * (2 * m + 2); }

void launch_step_kernels(const LsArgs& a, cudaStream_t s) {
  launch_pdl(k_ls_dots, dim3(a.G), dim3(kLT), dots_smem(a.m), s, a);
  count_launch();
  launch_pdl(k_ls_update, dim3(a.G2), dim3(kLT), update_smem(a.m), s, a);
  count_launch();
}

bool graph_mode_on() {
  static const bool on = [] {
    const char* v = std::getenv("MGRX_GMRES_GRAPH");
    return !(v && v[0] == '0');
  }();
  return on;
}

}  // namespace

void LsWork::ensure(int n_, int m_, cudaStream_t s) {
  if (n_ == n && m_ == m) return;
  n = n_;
  m = m_;
  ldv = (n + 31) / 32 * 32;
  G = device_sms();
  V.alloc(static_cast<size_t>(ldv) * (m + 1), s);
  U.alloc(n > 0 ? n : 1, s);
  part.alloc(static_cast<size_t>(2 * m + 2) * G, s);
  part2.alloc(2 * G, s);
  ticket.alloc(2, s);
  ticket.zero();
  st.alloc(1, s);
  dbl.alloc(static_cast<size_t>(2 * (m + 1) * m + 3 * m + 1 + 2 * m + 2 + m + 8), s);
  dbl.zero();
  rpart.alloc(2 * m + 2, s);
  gath.release();
  if (hst) cudaFreeHost(hst);
  MGRX_CK(cudaMallocHost(&hst, sizeof(LsState)));
  if (exec) cudaGraphExecDestroy(exec);
  exec = nullptr;
  exec_key = {};
}

LsWork::~LsWork() {
  if (hst) cudaFreeHost(hst);
  if (exec) cudaGraphExecDestroy(exec);
}

bool lowsync_supported(int n, int m) { return n >= 0 && m >= 1 && m <= kLsMaxRestart; }

// ---------------------------------------------------------------------------
// LsDriver: the host side of one low-sync GMRES, shared by the single-GPU
// solve and the sharded one (shard.cu).
LsDriver::LsDriver(LsWork& L, int n, int m, double* w) : L_(L), n_(n), m_(m), w_(w) {
  if (L_.n != n || L_.m != m) throw RuntimeError("LsDriver: work buffers not sized for this solve");
  args_ = std::make_unique<LsArgs>(make_args(L_, n, m, w));
}
LsDriver::~LsDriver() = default;
double* LsDriver::U() const { return L_.U.get(); }
const LsArgs& LsDriver::args() const { return *args_; }

void LsDriver::start_cycle(double bnorm, double target, int iters_left, cudaStream_t s) {
  LsState hs{};
  hs.bnorm = bnorm;
  hs.target = target;
  hs.iters_left = iters_left;
  *L_.hst = hs;
  MGRX_CK(cudaMemcpyAsync(L_.st.get(), L_.hst, sizeof(LsState), cudaMemcpyHostToDevice, s));
}

void LsDriver::step(cudaStream_t s) { launch_step_kernels(*args_, s); }

void LsDriver::step_sharded(int nranks, const Allgather& allgather, cudaStream_t s) {
  const int stride = 2 * m_ + 2;
  if (L_.gath.size() < static_cast<size_t>(nranks) * stride) L_.gath.alloc(static_cast<size_t>(nranks) * stride, s);
  LsArgs a = *args_;
  a.rank_part = L_.rpart.get();
  launch_pdl(k_ls_dots, dim3(a.G), dim3(kLT), dots_smem(m_), s, a);
  allgather(L_.rpart.get(), L_.gath.get(), stride, s);
  launch_pdl(k_ls_coef, dim3(1), dim3(kLT), dots_smem(m_), s, a, static_cast<const double*>(L_.gath.get()), nranks,
             stride);
  launch_pdl(k_ls_update, dim3(a.G2), dim3(kLT), update_smem(m_), s, a);
  allgather(L_.rpart.get(), L_.gath.get(), stride, s);
  launch_pdl(k_ls_finish, dim3(1), dim3(1), 0, s, a, static_cast<const double*>(L_.gath.get()), nranks, stride);
  count_launch(4);
}

const LsState& LsDriver::sync_state(cudaStream_t s) {
  MGRX_CK(cudaMemcpyAsync(L_.hst, L_.st.get(), sizeof(LsState), cudaMemcpyDeviceToHost, s));
  MGRX_CK(cudaStreamSynchronize(s));
  return *L_.hst;
}

// End of a restart cycle: the cycle's residual estimates (appended to
// hist) and the reference's triangular solve (krylov.cpp:119-124) on the
// rotated H (last column: its tentative rotation). Returns the state.
LsState LsDriver::end_cycle(std::vector<double>& hist, std::vector<double>& y, cudaStream_t s) {
  const LsState hs = sync_state(s);
  const int k = hs.steps;
  const LsArgs& a = *args_;
  std::vector<double> h(k), Hrot(static_cast<size_t>(m_ + 1) * m_), gv(m_ + 1);
  if (k > 0) MGRX_CK(cudaMemcpyAsync(h.data(), a.hist, sizeof(double) * k, cudaMemcpyDeviceToHost, s));
  MGRX_CK(cudaMemcpyAsync(Hrot.data(), a.Hrot, sizeof(double) * Hrot.size(), cudaMemcpyDeviceToHost, s));
  MGRX_CK(cudaMemcpyAsync(gv.data(), a.g, sizeof(double) * (m_ + 1), cudaMemcpyDeviceToHost, s));
  MGRX_CK(cudaStreamSynchronize(s));
  hist.insert(hist.end(), h.begin(), h.end());
  y.clear();
  if (k == 0 || (hs.flags & kLsNonFinite)) return hs;
  gv[k - 1] = hs.gt0;
  auto R = [&](int i, int j) { return Hrot[static_cast<size_t>(j) * (m_ + 1) + i]; };
  int keff = k;
  while (keff > 0 && std::abs(R(keff - 1, keff - 1)) < 1e-300) --keff;
  y.assign(keff, 0.0);
  for (int i = keff - 1; i >= 0; --i) {
    double acc = gv[i];
    for (int j = i + 1; j < keff; ++j) acc -= R(i, j) * y[j];
    y[i] = acc / R(i, i);
  }
  return hs;
}

void LsDriver::combine(const std::vector<double>& y, double* u, cudaStream_t s) {
  const int keff = static_cast<int>(y.size());
  const LsArgs& a = *args_;
  MGRX_CK(cudaMemcpyAsync(a.coef, y.data(), sizeof(double) * keff, cudaMemcpyHostToDevice, s));
  if (n_ > 0) {
    launch_pdl(k_ls_combine, dim3(blocks_for(n_, 256)), dim3(256), 0, s, n_, L_.ldv, keff,
               static_cast<const double*>(L_.V.get()), static_cast<const double*>(a.coef), u);
    count_launch();
  }
  MGRX_CK(cudaStreamSynchronize(s));  // y lives on the host
}

// Right-preconditioned restarted GMRES (proj/src/krylov.cpp:37-147) with the
// lagged CGS2 Arnoldi above. The restart-cycle work (triangular solve, x
// update, true residual) follows the reference's order on the host, reading
// the device's H, g and history once per cycle.
GmresResult gmres_lowsync(const DCsr& A, const double* b, double* x, const KrylovSpec& cfg, const DevOp& precond,
                          const DevOp& precond_capture, GmresWork& ws, cudaStream_t s) {
  NvtxRange nvtx("mgrx.gmres.cgs2");
  TeamSums team_sums(true);  // tolerance-level solve: SpMVs may use their team-sum kernels
  const int n = A.rows;
  const int m = cfg.restart;
  ws.ensure(n, 1, s);  // w, z, r, u, reduction scratch (MGS basis not needed)
  LsWork& L = ws.ls;
  L.ensure(n, m, s);
  double* w = ws.w.get();
  double* z = ws.z.get();
  LsDriver drv(L, n, m, w);
  double* U = drv.U();
  GmresResult res;
  auto prec = [&](const double* in, double* out) {
    if (precond) precond(in, out, s);
    else MGRX_CK(cudaMemcpyAsync(out, in, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  };
  auto norm2 = [&](const double* v) { return device_dot(n, v, v, ws, s); };

  const double bb = norm2(b);
  if (!std::isfinite(bb)) throw RuntimeError("gmres: rhs contains non-finite entries");
  const double bnorm = std::sqrt(bb);
  if (bnorm == 0.0) {
    MGRX_CK(cudaMemsetAsync(x, 0, sizeof(double) * n, s));
    res.converged = true;
    return res;
  }
  const double target = std::max(cfg.rel_tol * bnorm, cfg.abs_tol);

  // One restart cycle's steps as a CUDA graph: WHILE(!cycle_end) { M^-1, SpMV,
  // sweep A, sweep B }; the body's last kernel sets the condition.
  bool use_graph = graph_mode_on() && !L.graph_failed && (static_cast<bool>(precond_capture) || !precond);
  if (use_graph && (!L.exec || L.exec_key.w != w || L.exec_key.z != z || L.exec_key.A != &A)) {
    if (L.exec) cudaGraphExecDestroy(L.exec);
    L.exec = nullptr;
    cudaGraph_t g = nullptr;
    try {
      MGRX_CK(cudaGraphCreate(&g, 0));
      cudaGraphConditionalHandle h;
      MGRX_CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
      cudaGraphNodeParams np{};
      np.type = cudaGraphNodeTypeConditional;
      np.conditional.handle = h;
      np.conditional.type = cudaGraphCondTypeWhile;
      np.conditional.size = 1;
      cudaGraphNode_t node;
      MGRX_CK(cudaGraphAddNode(&node, g, nullptr, 0, &np));
      cudaGraph_t body = np.conditional.phGraph_out[0];
      LsArgs ag = drv.args();
      ag.cond = h;
      ag.use_cond = 1;
      const long long l0 = g_launches;
      MGRX_CK(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
      try {
        if (precond_capture) precond_capture(U, z, s);
        else MGRX_CK(cudaMemcpyAsync(z, U, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
        spmv(A, z, w, s);
        launch_step_kernels(ag, s);
      } catch (...) {
        cudaGraph_t dummy;
        cudaStreamEndCapture(s, &dummy);
        g_launches = l0;
        throw;
      }
      cudaGraph_t captured;
      MGRX_CK(cudaStreamEndCapture(s, &captured));
      L.body_nodes = g_launches - l0;
      g_launches = l0;
      MGRX_CK(cudaGraphInstantiate(&L.exec, g, 0));
      MGRX_CK(cudaGraphDestroy(g));
      g = nullptr;
      L.exec_key = {w, z, &A};
    } catch (const std::exception& e) {
      // conditional graphs unavailable here: host-driven steps (same kernels)
      if (g) cudaGraphDestroy(g);
      cudaGetLastError();
      if (std::getenv("MGRX_GMRES_GRAPH_DEBUG")) std::fprintf(stderr, "mgrx: cycle graph disabled: %s\n", e.what());
      L.graph_failed = true;
      L.exec = nullptr;
      use_graph = false;
    }
  }

  spmv_residual(A, x, b, nullptr, U, s);  // U = r = b - A x
  double rnorm = std::sqrt(norm2(U));
  std::vector<double> y;
  while (true) {
    if (!std::isfinite(rnorm)) throw RuntimeError("gmres: residual is non-finite");
    if (rnorm <= target) {
      res.converged = true;
      res.final_residual = rnorm / bnorm;
      res.history.push_back(res.final_residual);
      return res;
    }
    if (res.iterations >= cfg.max_iters) {
      res.final_residual = rnorm / bnorm;
      return res;
    }
    // the cycle starts from U = r (v_0 = r / ||r|| in sweep B)
    drv.start_cycle(bnorm, target, std::min(m, cfg.max_iters - res.iterations), s);
    if (use_graph) {
      MGRX_CK(cudaGraphLaunch(L.exec, s));
      count_launch(L.body_nodes * drv.sync_state(s).steps);
    } else {
      do {
        prec(U, z);
        spmv(A, z, w, s);
        drv.step(s);
      } while (!(drv.sync_state(s).flags & kLsCycleEnd));
    }
    const LsState hs = drv.end_cycle(res.history, y, s);
    if (hs.flags & kLsNonFinite) throw RuntimeError("gmres: Arnoldi vector is non-finite");
    res.iterations += hs.steps;
    if (!y.empty()) {
      drv.combine(y, ws.u.get(), s);
      prec(ws.u.get(), z);
      vec_add(n, z, x, s);  // x += M^{-1}(V y)
    }
    spmv_residual(A, x, b, nullptr, U, s);
    const double tn = std::sqrt(norm2(U));
    if (!std::isfinite(tn)) throw RuntimeError("gmres: residual is non-finite");
    res.history.push_back(tn / bnorm);
    if (tn <= target) {
      res.converged = true;
      res.final_residual = tn / bnorm;
      return res;
    }
    if (hs.flags & kLsHappy) throw RuntimeError("gmres: Arnoldi breakdown before reaching tolerance");
    res.final_residual = tn / bnorm;
    if (res.iterations >= cfg.max_iters) return res;
    rnorm = tn;  // the next cycle starts from this residual (already in U)
  }
}

// Probe (bench roofline): one step's two sweeps at step index k on the work
// vectors (U, w hold whatever the last solve left; values do not matter).
int lowsync_probe(int n, int k, GmresWork& ws, cudaStream_t s, int which) {
  const int m = 30;
  if (k < 0 || k >= m) return 0;
  ws.ensure(n, 1, s);
  LsWork& L = ws.ls;
  L.ensure(n, m, s);
  LsArgs a = make_args(L, n, m, ws.w.get());
  LsState hs{};
  hs.k = k;
  hs.bnorm = 1.0;
  hs.iters_left = m;
  *L.hst = hs;
  MGRX_CK(cudaMemcpyAsync(L.st.get(), L.hst, sizeof(LsState), cudaMemcpyHostToDevice, s));
  if (which & 1) {
    launch_pdl(k_ls_dots, dim3(a.G), dim3(kLT), dots_smem(m), s, a);
    count_launch();
  }
  if (which & 2) {
    launch_pdl(k_ls_update, dim3(a.G2), dim3(kLT), update_smem(m), s, a);
    count_launch();
  }
  return 1;
}

}  // namespace mgrx
