// Smoother kernels. The Gauss-Seidel sweep is the reference's sequential
// loop (proj/src/relax.cpp:55-78, one range) executed sync-free: rows are
// dispatched in dependency-level order through a ticket counter, and each
// row polls the values it depends on. A value doubles as its own ready flag:
// xnew is pre-filled with an all-ones NaN pattern that no finite result can
// produce, and a finished row publishes its 64-bit result with one relaxed
// gpu-scope store. Every row performs exactly the reference's operations in
// the reference's order, so the result is bitwise equal to the CPU loop.
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "relax.cuh"

namespace mgrx {
namespace {

constexpr int kGsThreads = 128;
constexpr int kGsCap = 4096;  // sweep-CSR entries staged in shared memory per CTA
constexpr size_t kGsSmem = kGsCap * (2 * sizeof(double) + sizeof(int));
#ifndef MGRX_KPOLL
#define MGRX_KPOLL 8
#endif
constexpr int kPoll = MGRX_KPOLL;  // entries polled per lane per round
constexpr long long kSpinLimit = 1LL << 24;
constexpr int kDepBit = 1 << 31;

__device__ __forceinline__ double ld_relaxed(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_relaxed(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v));
}
__device__ __forceinline__ int ld_relaxed_int(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ bool pending_value(double v) { return __double_as_longlong(v) == -1LL; }

// Optional sweep trace (MGRX_GS_TRACE=<dir>): per row, the %globaltimer when
// its lane started on it and when it published x_i. Diagnostic only.
__device__ unsigned long long* g_trace_start = nullptr;
__device__ unsigned long long* g_trace_pub = nullptr;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Sync-free sweep kernel. A team of kT lanes owns one row (kT = 1, 4 or 8,
// chosen from the average dependency count). The CTA takes kGsThreads/kT
// consecutive sweep positions per ticket and stages their sweep-CSR entries
// in shared memory, next to one value slot per entry. In every round the team
// lanes poll all still-missing dependency values of the row in parallel and
// park them in the slots; the team leader folds the slots into the row sum in
// stored order for as far as they are filled. So when the last dependency
// lands, everything else is already on chip and the row finishes at once.
// kFull: entries carry a dependency flag; other columns read the old iterate.
// Persistent CTAs: the grid keeps only a few dependency levels in flight, so
// polling does not starve the rows that produce values.
template <int kT, bool kFull>
__global__ void __launch_bounds__(kGsThreads)
    k_gs(int n, const int* __restrict__ order, const int* __restrict__ sptr,
         const int* __restrict__ scol, const double* __restrict__ sval, const double* __restrict__ sd,
         const double* __restrict__ b, const double* __restrict__ xold, double* xnew, double* zadd,
         int* tk, unsigned sleep_ns, int pub_mode) {
  extern __shared__ double smem[];
  double* cval = smem;                     // kGsCap entry values
  double* cx = smem + kGsCap;              // kGsCap parked x values
  int* ccol = reinterpret_cast<int*>(smem + 2 * kGsCap);
  __shared__ int base;
  constexpr int kRowsPerCta = kGsThreads / kT;
  const int lane = threadIdx.x & 31;
  const int u = lane % kT;                 // lane within team
  const int leader = lane - u;
  const unsigned team_mask = (kT == 32 ? 0xffffffffu : ((1u << kT) - 1u)) << leader;
  while (true) {
    if (threadIdx.x == 0) base = atomicAdd(tk, kRowsPerCta);
    __syncthreads();
    const int p0 = base;
    if (p0 >= n) return;
    const int pend = min(p0 + kRowsPerCta, n);
    const int e0 = sptr[p0], e1 = sptr[pend];
    const bool staged = (e1 - e0) <= kGsCap;
    if (staged)
      for (int q = e0 + threadIdx.x; q < e1; q += kGsThreads) {
        int c = scol[q];
        ccol[q - e0] = c;
        cval[q - e0] = sval[q];
        double v = __longlong_as_double(-1LL);
        if (kFull && !(c & kDepBit)) v = xold[c];
        cx[q - e0] = v;
      }
    __syncthreads();
    const int p = p0 + threadIdx.x / kT;
    const bool active = p < n;
    int i = 0, k = 0, ke = 0;
    double s = 0.0;
    if (active) {
      i = order[p];
      k = sptr[p];
      ke = sptr[p + 1];
      if (u == 0) s = b[i];
      if (g_trace_start && u == 0) g_trace_start[i] = gtimer();
    }
    bool done = !active;
    long long spins = 0;
    while (!__all_sync(0xffffffffu, done)) {
      if (!done) {
        if (staged) {
          // poll the missing dependencies of the row's next kPoll*kT entries
          // (team-strided): all loads are issued before any is consumed, so a
          // round costs one L2 round trip however many values are missing
          bool need[kPoll];
          int ce[kPoll];
          double pv[kPoll];
#pragma unroll
          for (int t = 0; t < kPoll; ++t) {
            const int e = k + u + t * kT;
            need[t] = e < ke && pending_value(cx[e - e0]);
            int c = need[t] ? ccol[e - e0] : 0;
            if (kFull) c &= ~kDepBit;
            ce[t] = c;
          }
#pragma unroll
          for (int t = 0; t < kPoll; ++t)
            if (need[t]) pv[t] = ld_relaxed(xnew + ce[t]);
#pragma unroll
          for (int t = 0; t < kPoll; ++t)
            if (need[t] && !pending_value(pv[t])) cx[k + u + t * kT - e0] = pv[t];
          __syncwarp(team_mask);
          int k2 = k;
          if (u == 0) {
            while (k2 < ke && !pending_value(cx[k2 - e0])) {
              s = __dsub_rn(s, __dmul_rn(cval[k2 - e0], cx[k2 - e0]));
              ++k2;
            }
          }
          k2 = __shfl_sync(team_mask, k2, leader);
          const bool progressed = k2 > k;
          k = k2;
          if (k >= ke) {
            if (u == 0) {
              const double xi = kFull ? xold[i] : 0.0;
              const double v = __dadd_rn(xi, __ddiv_rn(s, sd[p]));
              if (pub_mode == 2) {
                atomicExch(reinterpret_cast<unsigned long long*>(xnew + i),
                           static_cast<unsigned long long>(__double_as_longlong(v)));
              } else {
                st_relaxed(xnew + i, v);
                if (pub_mode == 1) asm volatile("fence.acq_rel.gpu;" ::: "memory");
              }
              if (g_trace_pub) g_trace_pub[i] = gtimer();
              if (zadd) zadd[i] = __dadd_rn(zadd[i], v);
            }
            done = true;
          } else if (!progressed) {
            if (++spins > kSpinLimit) {
              if (u == 0) {
                atomicExch(tk + 1, 1);
                st_relaxed(xnew + i, 0.0);
              }
              done = true;
            } else if (sleep_ns > 0) {
              __nanosleep(sleep_ns);
            }
          }
        } else {
          // unstaged fallback (huge rows): leader walks the row from global memory
          bool prog = false;
          if (u == 0) {
            while (k < ke) {
              int c = scol[k];
              double xv;
              if (kFull && !(c & kDepBit)) {
                xv = xold[c];
              } else {
                if (kFull) c &= ~kDepBit;
                xv = ld_relaxed(xnew + c);
                if (pending_value(xv)) break;
              }
              s = __dsub_rn(s, __dmul_rn(sval[k], xv));
              ++k;
              prog = true;
            }
          }
          k = __shfl_sync(team_mask, k, leader);
          prog = __shfl_sync(team_mask, prog, leader);
          if (k >= ke) {
            if (u == 0) {
              const double xi = kFull ? xold[i] : 0.0;
              const double v = __dadd_rn(xi, __ddiv_rn(s, sd[p]));
              st_relaxed(xnew + i, v);
              if (zadd) zadd[i] = __dadd_rn(zadd[i], v);
            }
            done = true;
          } else if (!prog) {
            if (++spins > kSpinLimit) {
              if (u == 0) {
                atomicExch(tk + 1, 1);
                st_relaxed(xnew + i, 0.0);
              }
              done = true;
            } else {
              __nanosleep(20);
            }
          }
        }
      }
    }
    __syncthreads();
  }
}

// Level-synchronous sweep inside one thread-block cluster: all CTAs of the
// cluster walk the dependency levels in lockstep; rows of a level are
// independent, so each thread computes whole rows (same arithmetic, same
// order), publishes x_i to L2 (st.cg), and a cluster barrier (release /
// acquire) separates levels. Reads of new values bypass L1 (ld.cg), so no SM
// sees a stale line. Latency hiding: a thread's row for level L+1 (indices,
// rhs, diagonal and up to kLvChunk entries) is loaded into registers before
// the barrier that ends level L, and all its dependency values are then
// requested at once, so a level costs about one L2 round trip plus the
// barrier instead of a chain of dependent loads.
constexpr int kLvThreads = 512;
constexpr int kLvChunk = 8;
constexpr int kLvMaxLevels = 8192;

template <bool kFull, bool kCluster>
__global__ void __launch_bounds__(kLvThreads)
    k_gs_lv(int nlev, const int* __restrict__ lptr, const int* __restrict__ order,
            const int* __restrict__ sptr, const int* __restrict__ scol, const double* __restrict__ sval,
            const double* __restrict__ sd, const double* __restrict__ b, const double* __restrict__ xold,
            double* xnew, double* zadd) {
  namespace cg = cooperative_groups;
  __shared__ int slp[kLvMaxLevels + 1];
  int nthr = blockDim.x, tid = threadIdx.x;
  if (kCluster) {
    cg::cluster_group cl = cg::this_cluster();
    nthr = static_cast<int>(cl.num_blocks()) * blockDim.x;
    tid = static_cast<int>(cl.block_rank()) * blockDim.x + threadIdx.x;
  }
  const bool lp_smem = nlev <= kLvMaxLevels;
  if (lp_smem)
    for (int q = threadIdx.x; q <= nlev; q += blockDim.x) slp[q] = lptr[q];
  __syncthreads();
#define LP(q) (lp_smem ? slp[(q)] : lptr[(q)])
  // register-resident prefetched row
  int ri = 0, rk0 = 0, rk1 = 0, rp = 0;
  double rb = 0.0, rd = 1.0;
  int rc[kLvChunk];
  double ra[kLvChunk];
  bool have = false;
#define LV_FETCH(P)                                                    \
  {                                                                    \
    rp = (P);                                                          \
    ri = order[rp];                                                    \
    rk0 = sptr[rp];                                                    \
    rk1 = sptr[rp + 1];                                                \
    rb = b[ri];                                                        \
    rd = sd[rp];                                                       \
    const int m_ = rk1 - rk0;                                          \
    _Pragma("unroll") for (int q = 0; q < kLvChunk; ++q) if (q < m_) { \
      rc[q] = scol[rk0 + q];                                           \
      ra[q] = sval[rk0 + q];                                           \
    }                                                                  \
  }
#define LV_XLOAD(C, OUT)                   \
  {                                        \
    int c_ = (C);                          \
    if (kFull && !(c_ & kDepBit)) {        \
      OUT = xold[c_];                      \
    } else {                               \
      if (kFull) c_ &= ~kDepBit;           \
      OUT = __ldcg(xnew + c_);             \
    }                                      \
  }
#define LV_ROW()                                                                  \
  {                                                                               \
    double s_ = rb;                                                               \
    const int m_ = rk1 - rk0;                                                     \
    double xv_[kLvChunk];                                                         \
    _Pragma("unroll") for (int q = 0; q < kLvChunk; ++q) if (q < m_)              \
        LV_XLOAD(rc[q], xv_[q]);                                                  \
    _Pragma("unroll") for (int q = 0; q < kLvChunk; ++q) if (q < m_)              \
        s_ = __dsub_rn(s_, __dmul_rn(ra[q], xv_[q]));                             \
    for (int k0 = rk0 + kLvChunk; k0 < rk1; k0 += kLvChunk) {                     \
      const int mm_ = min(kLvChunk, rk1 - k0);                                    \
      _Pragma("unroll") for (int q = 0; q < kLvChunk; ++q) if (q < mm_) {         \
        rc[q] = scol[k0 + q];                                                     \
        ra[q] = sval[k0 + q];                                                     \
      }                                                                           \
      _Pragma("unroll") for (int q = 0; q < kLvChunk; ++q) if (q < mm_)           \
          LV_XLOAD(rc[q], xv_[q]);                                                \
      _Pragma("unroll") for (int q = 0; q < kLvChunk; ++q) if (q < mm_)           \
          s_ = __dsub_rn(s_, __dmul_rn(ra[q], xv_[q]));                           \
    }                                                                             \
    const double v_ = __dadd_rn(kFull ? xold[ri] : 0.0, __ddiv_rn(s_, rd));       \
    __stcg(xnew + ri, v_);                                                        \
    if (zadd) zadd[ri] = __dadd_rn(zadd[ri], v_);                                 \
  }
  {
    const int p = LP(0) + tid;
    if (p < LP(1)) {
      LV_FETCH(p);
      have = true;
    }
  }
  for (int L = 0; L < nlev; ++L) {
    const int e = LP(L + 1);
    if (have) LV_ROW();
    for (int p = LP(L) + tid + nthr; p < e; p += nthr) {
      LV_FETCH(p);
      LV_ROW();
    }
    have = false;
    if (L + 1 < nlev) {
      const int p = e + tid;
      if (p < LP(L + 2)) {
        LV_FETCH(p);
        have = true;
      }
    }
    if (kCluster) {
      cg::this_cluster().sync();
    } else {
      __syncthreads();
    }
  }
#undef LP
#undef LV_FETCH
#undef LV_XLOAD
#undef LV_ROW
}

// Pipelined single-CTA level sweep. The sweep is cut into "steps": runs of
// consecutive sweep positions inside one dependency level that fit a shared
// memory buffer (kPipeRows rows, kPipeEnt entries). One 1024-thread CTA walks
// the steps; while it computes step s it prefetches step s+1 (row ids, rhs in
// sweep order, diagonal, dependency columns/values) with cp.async into the
// other buffer, so a step costs the L2 round trip of its x values plus a
// barrier. Rows in a step are independent; values are published with st.cg
// and read with ld.cg, ordered by __syncthreads inside the CTA.
constexpr int kPipeThreads = 1024;
constexpr int kPipeRows = 1536;
constexpr int kPipeEnt = 5120;
struct PipeBuf {
  double sd[kPipeRows];
  double bp[kPipeRows];
  double val[kPipeEnt];
  int ord[kPipeRows];
  int ptr[kPipeRows + 1];
  int col[kPipeEnt];
};
constexpr size_t kPipeSmem = 2 * sizeof(PipeBuf);
constexpr int kPipeMaxSteps = 2048;

__device__ __forceinline__ void cpa4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
               "l"(src));
}
__device__ __forceinline__ void cpa8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
               "l"(src));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;"); }
__device__ __forceinline__ void cpa_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

template <bool kFull>
__global__ void __launch_bounds__(kPipeThreads)
    k_gs_pipe(int nsteps, const int* __restrict__ steps, const int* __restrict__ order,
              const int* __restrict__ sptr, const int* __restrict__ scol, const double* __restrict__ sval,
              const double* __restrict__ sd, const double* __restrict__ bp, const double* __restrict__ xold,
              double* xnew, double* zadd) {
  extern __shared__ __align__(16) unsigned char pipe_raw[];
  PipeBuf* buf = reinterpret_cast<PipeBuf*>(pipe_raw);
  const int tid = threadIdx.x;
  // step boundaries (positions and entry offsets) staged once, so issuing a
  // prefetch never waits on a global load
  __shared__ int stp[kPipeMaxSteps + 1], ste[kPipeMaxSteps + 1];
  const bool st_smem = nsteps <= kPipeMaxSteps;
  if (st_smem)
    for (int q = tid; q <= nsteps; q += kPipeThreads) {
      stp[q] = steps[q];
      ste[q] = steps[nsteps + 1 + q];
    }
  __syncthreads();
  auto SP = [&](int q) { return st_smem ? stp[q] : steps[q]; };
  auto SE = [&](int q) { return st_smem ? ste[q] : steps[nsteps + 1 + q]; };
  auto issue = [&](int st, PipeBuf& B) {
    const int p0 = SP(st), p1 = SP(st + 1);
    const int nr = p1 - p0;
    const int e0 = SE(st), e1 = SE(st + 1);
    for (int q = tid; q < nr; q += kPipeThreads) {
      cpa4(&B.ord[q], order + p0 + q);
      cpa8(&B.sd[q], sd + p0 + q);
      cpa8(&B.bp[q], bp + p0 + q);
    }
    for (int q = tid; q <= nr; q += kPipeThreads) cpa4(&B.ptr[q], sptr + p0 + q);
    for (int q = tid; q < e1 - e0; q += kPipeThreads) {
      cpa4(&B.col[q], scol + e0 + q);
      cpa8(&B.val[q], sval + e0 + q);
    }
    cpa_commit();
  };
  issue(0, buf[0]);
  for (int st = 0; st < nsteps; ++st) {
    PipeBuf& B = buf[st & 1];
    if (st + 1 < nsteps) issue(st + 1, buf[(st + 1) & 1]);
    else cpa_commit();  // keep the group count uniform for wait_group 1
    cpa_wait1();
    __syncthreads();
    const int nr = SP(st + 1) - SP(st);
    const int e0 = B.ptr[0];
    for (int q = tid; q < nr; q += kPipeThreads) {
      const int i = B.ord[q];
      double s = B.bp[q];
      const int k1 = B.ptr[q + 1] - e0;
      for (int k = B.ptr[q] - e0; k < k1; ++k) {
        int c = B.col[k];
        double x;
        if (kFull && !(c & kDepBit)) {
          x = xold[c];
        } else {
          if (kFull) c &= ~kDepBit;
          x = __ldcg(xnew + c);
        }
        s = __dsub_rn(s, __dmul_rn(B.val[k], x));
      }
      const double v = __dadd_rn(kFull ? xold[i] : 0.0, __ddiv_rn(s, B.sd[q]));
      __stcg(xnew + i, v);
      if (zadd) zadd[i] = __dadd_rn(zadd[i], v);
    }
    __syncthreads();
  }
}

__global__ void k_gather_d(int n, const int* __restrict__ idx, const double* __restrict__ x,
                           double* __restrict__ y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = x[idx[i]];
}

// Small-level variant: the whole iterate x lives in shared memory (n <=
// kSmallN), so a dependency level costs shared-memory latency plus one
// barrier — no L2 round trip on the critical path. Row data streams through
// two cp.async buffers exactly as in k_gs_pipe. This is what the coarse AMG
// levels use (their dependency chains are long: 343 / 160 / 59 levels at cfg2).
constexpr int kSmallN = 12288;
constexpr int kSmallRows = 512;
constexpr int kSmallEnt = 2048;
struct SmallBuf {
  double sd[kSmallRows];
  double bp[kSmallRows];
  double val[kSmallEnt];
  int ord[kSmallRows];
  int ptr[kSmallRows + 1];
  int col[kSmallEnt];
};
constexpr size_t kSmallSmem = 2 * sizeof(SmallBuf) + kSmallN * sizeof(double);

template <bool kFull>
__global__ void __launch_bounds__(kPipeThreads)
    k_gs_small(int nsteps, const int* __restrict__ steps, int nchunks, const int* __restrict__ chunks,
               const int* __restrict__ order,
               const int* __restrict__ sptr, const int* __restrict__ scol, const double* __restrict__ sval,
               const double* __restrict__ sd, const double* __restrict__ bp, const double* __restrict__ xold,
               double* xnew, double* zadd) {
  extern __shared__ __align__(16) unsigned char small_raw[];
  SmallBuf* buf = reinterpret_cast<SmallBuf*>(small_raw);
  double* xs = reinterpret_cast<double*>(small_raw + 2 * sizeof(SmallBuf));
  const int tid = threadIdx.x;
  __shared__ int stp[kPipeMaxSteps + 1], ste[kPipeMaxSteps + 1];
  const bool st_smem = nsteps <= kPipeMaxSteps;
  if (st_smem)
    for (int q = tid; q <= nsteps; q += kPipeThreads) {
      stp[q] = steps[q];
      ste[q] = steps[nsteps + 1 + q];
    }
  __syncthreads();
  auto SP = [&](int q) { return st_smem ? stp[q] : steps[q]; };
  auto SE = [&](int q) { return st_smem ? ste[q] : steps[nsteps + 1 + q]; };
  // chunk c = steps [chunks[c], chunks[c+1]): its rows and entries are
  // contiguous, loaded by one cp.async group while the previous chunk's
  // dependency levels are swept (one barrier per level)
  auto issue = [&](int c, SmallBuf& B) {
    const int sa = chunks[c], sb = chunks[c + 1];
    const int p0 = SP(sa), p1 = SP(sb);
    const int nr = p1 - p0;
    const int e0 = SE(sa), e1 = SE(sb);
    for (int q = tid; q < nr; q += kPipeThreads) {
      cpa4(&B.ord[q], order + p0 + q);
      cpa8(&B.sd[q], sd + p0 + q);
      cpa8(&B.bp[q], bp + p0 + q);
    }
    for (int q = tid; q <= nr; q += kPipeThreads) cpa4(&B.ptr[q], sptr + p0 + q);
    for (int q = tid; q < e1 - e0; q += kPipeThreads) {
      cpa4(&B.col[q], scol + e0 + q);
      cpa8(&B.val[q], sval + e0 + q);
    }
    cpa_commit();
  };
  (void)nsteps;
  issue(0, buf[0]);
  for (int c = 0; c < nchunks; ++c) {
    SmallBuf& B = buf[c & 1];
    if (c + 1 < nchunks) issue(c + 1, buf[(c + 1) & 1]);
    else cpa_commit();
    cpa_wait1();
    __syncthreads();
    const int cbase = SP(chunks[c]);
    for (int st = chunks[c]; st < chunks[c + 1]; ++st) {
    const int qa = SP(st) - cbase, qb = SP(st + 1) - cbase;
    const int e0 = B.ptr[0];
    for (int q = qa + tid; q < qb; q += kPipeThreads) {
      const int i = B.ord[q];
      double s = B.bp[q];
      const int k1 = B.ptr[q + 1] - e0;
      // operand loads of 4 entries are issued together (the column index and
      // the iterate value are dependent shared-memory loads; one entry at a
      // time the row was bound by their latency), then the entries are
      // subtracted in the row's order
      auto xval = [&](int c) -> double {
        if (kFull && !(c & kDepBit)) return xold[c];
        return xs[kFull ? (c & ~kDepBit) : c];
      };
      int k = B.ptr[q] - e0;
      for (; k + 4 <= k1; k += 4) {
        const int c0 = B.col[k], c1 = B.col[k + 1], c2 = B.col[k + 2], c3 = B.col[k + 3];
        const double x0 = xval(c0), x1 = xval(c1), x2 = xval(c2), x3 = xval(c3);
        const double p0 = __dmul_rn(B.val[k], x0), p1 = __dmul_rn(B.val[k + 1], x1);
        const double p2 = __dmul_rn(B.val[k + 2], x2), p3 = __dmul_rn(B.val[k + 3], x3);
        s = __dsub_rn(__dsub_rn(__dsub_rn(__dsub_rn(s, p0), p1), p2), p3);
      }
      for (; k < k1; ++k) s = __dsub_rn(s, __dmul_rn(B.val[k], xval(B.col[k])));
      const double v = __dadd_rn(kFull ? xold[i] : 0.0, __ddiv_rn(s, B.sd[q]));
      xs[i] = v;
      xnew[i] = v;
      if (zadd) zadd[i] = __dadd_rn(zadd[i], v);
    }
    __syncthreads();
    }
  }
}

// Block-partitioned sweep from zero (dep-only entries). A CTA takes the next
// row block (processing order) from a ticket counter, so every block it
// waits on was taken earlier by a running CTA (deadlock-free). The block's
// rows are swept in local dependency-level order with its iterate in shared
// memory (xs, indexed by row - lo), chunks of steps double-buffered by
// cp.async exactly as in k_gs_small. Entries flagged kCrossBit depend on an
// earlier block: the value is polled from xnew (pre-filled with the pending
// pattern; published with one relaxed 64-bit store). Per row: the
// reference's operations in its order (bitwise equal).
constexpr int kCrossBit = 1 << 30;
__global__ void __launch_bounds__(kPipeThreads)
    k_gs_blk(int nblk, const int* __restrict__ blk_lo, const int* __restrict__ blk_chunk,
             int nsteps, const int* __restrict__ steps, const int* __restrict__ chunks,
             const int* __restrict__ order, const int* __restrict__ sptr, const int* __restrict__ scol,
             const double* __restrict__ sval, const double* __restrict__ sd, const double* __restrict__ bp,
             double* xnew, double* zadd, int* tk) {
  extern __shared__ __align__(16) unsigned char blk_raw[];
  SmallBuf* buf = reinterpret_cast<SmallBuf*>(blk_raw);
  double* xs = reinterpret_cast<double*>(blk_raw + 2 * sizeof(SmallBuf));
  const int tid = threadIdx.x;
  __shared__ int bidx;
  auto SP = [&](int q) { return steps[q]; };
  auto SE = [&](int q) { return steps[nsteps + 1 + q]; };
  auto issue = [&](int c, SmallBuf& B) {
    const int sa = chunks[c], sb = chunks[c + 1];
    const int p0 = SP(sa), p1 = SP(sb);
    const int nr = p1 - p0;
    const int e0 = SE(sa), e1 = SE(sb);
    for (int q = tid; q < nr; q += kPipeThreads) {
      cpa4(&B.ord[q], order + p0 + q);
      cpa8(&B.sd[q], sd + p0 + q);
      cpa8(&B.bp[q], bp + p0 + q);
    }
    for (int q = tid; q <= nr; q += kPipeThreads) cpa4(&B.ptr[q], sptr + p0 + q);
    for (int q = tid; q < e1 - e0; q += kPipeThreads) {
      cpa4(&B.col[q], scol + e0 + q);
      cpa8(&B.val[q], sval + e0 + q);
    }
    cpa_commit();
  };
  while (true) {
    if (tid == 0) bidx = atomicAdd(tk, 1);
    __syncthreads();
    const int bk = bidx;
    if (bk >= nblk) return;
    const int lo = blk_lo[bk];
    const int c0 = blk_chunk[bk], c1 = blk_chunk[bk + 1];
    issue(c0, buf[0]);
    for (int c = c0; c < c1; ++c) {
      SmallBuf& B = buf[(c - c0) & 1];
      if (c + 1 < c1) issue(c + 1, buf[(c + 1 - c0) & 1]);
      else cpa_commit();
      cpa_wait1();
      __syncthreads();
      const int cbase = SP(chunks[c]);
      for (int st = chunks[c]; st < chunks[c + 1]; ++st) {
        const int qa = SP(st) - cbase, qb = SP(st + 1) - cbase;
        const int e0 = B.ptr[0];
        for (int q = qa + tid; q < qb; q += kPipeThreads) {
          const int i = B.ord[q];
          double s = B.bp[q];
          const int k1 = B.ptr[q + 1] - e0;
          auto xval = [&](int cc) -> double {
            if (!(cc & kCrossBit)) return xs[cc];
            const double* p = xnew + (cc & ~kCrossBit);
            double v = ld_relaxed(p);
            long long spins = 0;
            while (pending_value(v)) {
              if (++spins > kSpinLimit) {
                atomicExch(tk + 1, 1);
                return 0.0;
              }
              __nanosleep(32);
              v = ld_relaxed(p);
            }
            return v;
          };
          int k = B.ptr[q] - e0;
          for (; k + 4 <= k1; k += 4) {
            const int cc0 = B.col[k], cc1 = B.col[k + 1], cc2 = B.col[k + 2], cc3 = B.col[k + 3];
            const double x0 = xval(cc0), x1 = xval(cc1), x2 = xval(cc2), x3 = xval(cc3);
            const double p0 = __dmul_rn(B.val[k], x0), p1 = __dmul_rn(B.val[k + 1], x1);
            const double p2 = __dmul_rn(B.val[k + 2], x2), p3 = __dmul_rn(B.val[k + 3], x3);
            s = __dsub_rn(__dsub_rn(__dsub_rn(__dsub_rn(s, p0), p1), p2), p3);
          }
          for (; k < k1; ++k) s = __dsub_rn(s, __dmul_rn(B.val[k], xval(B.col[k])));
          const double v = __dadd_rn(0.0, __ddiv_rn(s, B.sd[q]));
          xs[i - lo] = v;
          st_relaxed(xnew + i, v);
          if (zadd) zadd[i] = __dadd_rn(zadd[i], v);
        }
        __syncthreads();
      }
    }
    __syncthreads();  // buffers and xs are reused by the next block
  }
}

// Group consecutive sweep steps into chunks of <= rows_cap rows / ent_cap
// entries (st: step row boundaries, ptr: the sweep CSR's row pointer).
std::vector<int> small_chunks(const std::vector<int>& st, const std::vector<int>& ptr, int rows_cap, int ent_cap) {
  std::vector<int> ch{0};
  const int ns = static_cast<int>(st.size()) - 1;
  int a = 0;
  while (a < ns) {
    int b = a + 1;
    while (b < ns && st[b + 1] - st[a] <= rows_cap && ptr[st[b + 1]] - ptr[st[a]] <= ent_cap) ++b;
    ch.push_back(b);
    a = b;
  }
  return ch;
}

std::vector<int> pipe_steps(const std::vector<int>& level_ptr, const std::vector<int>& sptr,
                            int rows_cap = kPipeRows, int ent_cap = kPipeEnt) {
  std::vector<int> st{0};
  for (size_t L = 0; L + 1 < level_ptr.size(); ++L) {
    int p = level_ptr[L];
    const int pe = level_ptr[L + 1];
    while (p < pe) {
      int q = p;
      while (q < pe && q - p < rows_cap && sptr[q + 1] - sptr[p] <= ent_cap) ++q;
      if (q == p) ++q;  // a single row longer than the buffer is never produced by the generators
      st.push_back(q);
      p = q;
    }
  }
  return st;
}

// Dependency levels by monotone in-place relaxation: lev[i] = 1 + max over
// dependencies; converges to the longest-path level.
// Dependency test of a sweep: j is visited before i in i's own range
// (hybrid partitions, proj/src/relax.cpp:68-73: other ranges read the
// snapshot). owner == nullptr: one range.
__device__ __forceinline__ bool is_dep(int i, int j, int fwd, const int* __restrict__ owner) {
  return (fwd ? (j < i) : (j > i)) && (owner == nullptr || owner[j] == owner[i]);
}
__global__ void k_levels(int n, const int* __restrict__ ptr, const int* __restrict__ col, int fwd,
                         const int* __restrict__ owner, int* lev, int* changed) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int m = 0;
  for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
    const int j = col[k];
    if (is_dep(i, j, fwd, owner)) {
      const int l = ld_relaxed_int(lev + j) + 1;
      m = l > m ? l : m;
    }
  }
  if (m > lev[i]) {
    lev[i] = m;
    *changed = 1;
  }
}
__global__ void k_iota(int n, int* a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = i;
}
// Sweep CSR construction (positions p in sweep order).
__global__ void k_sweep_count(int n, const int* __restrict__ order, const int* __restrict__ ptr,
                              const int* __restrict__ col, int fwd, const int* __restrict__ owner, int full,
                              int* __restrict__ cnt) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int i = order[p];
  int c = 0;
  for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
    const int j = col[k];
    c += (full || is_dep(i, j, fwd, owner)) ? 1 : 0;
  }
  cnt[p] = c;
}
__global__ void k_sweep_fill(int n, const int* __restrict__ order, const int* __restrict__ ptr,
                             const int* __restrict__ col, const double* __restrict__ val, int fwd,
                             const int* __restrict__ owner, int full, const int* __restrict__ sptr,
                             int* __restrict__ scol, double* __restrict__ sval) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int i = order[p];
  int o = sptr[p];
  for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
    const int j = col[k];
    const bool dep = is_dep(i, j, fwd, owner);
    if (!full && !dep) continue;
    scol[o] = (full && dep) ? (j | kDepBit) : j;
    sval[o] = val[k];
    ++o;
  }
}
__global__ void k_jacobi0(int n, double w, const double* __restrict__ dinv,
                          const double* __restrict__ r, const int* __restrict__ rrow,
                          double* __restrict__ z) {
  pdl_enter();
  // two elements per thread (i and i + 256, both coalesced): the gathered
  // form is a chain index -> value, so the second element's loads double
  // the requests in flight
  const int i = blockIdx.x * 512 + threadIdx.x, j = i + 256;
  if (i >= n) return;
  const bool vj = j < n;
  const int qi = rrow ? rrow[i] : i, qj = vj ? (rrow ? rrow[j] : j) : 0;
  const double di = dinv[i], dj = vj ? dinv[j] : 0.0;
  const double ri = r[qi], rj = vj ? r[qj] : 0.0;
  z[i] = __dmul_rn(w, __dmul_rn(di, ri));
  if (vj) z[j] = __dmul_rn(w, __dmul_rn(dj, rj));
}
__global__ void k_vec_add(int n, const double* __restrict__ a, double* __restrict__ y) {
  pdl_enter();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = __dadd_rn(y[i], a[i]);
}
__global__ void k_gather(int n, const int* __restrict__ idx, const double* __restrict__ x,
                         double* __restrict__ y) {
  pdl_enter();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = x[idx[i]];
}
__global__ void k_recip(int n, const double* __restrict__ d, double* __restrict__ y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = __ddiv_rn(1.0, d[i]);
}

void build_sweep_csr(const DCsr& A, const GsSchedule& sch, bool forward, const int* owner, bool full,
                     DVec<int>& sptr, DVec<int>& scol, DVec<double>& sval, cudaStream_t s) {
  const int n = A.rows;
  DVec<int> cnt(n, s);
  sptr.alloc(n + 1, s);
  const int nb = blocks_for(n, 256);
  k_sweep_count<<<nb, 256, 0, s>>>(n, sch.order.get(), A.ptr.get(), A.col.get(), forward ? 1 : 0,
                                   owner, full ? 1 : 0, cnt.get());
  MGRX_LAUNCH_CK();
  count_launch();
  const int nnz = static_cast<int>(exclusive_scan(cnt.get(), sptr.get(), n, s));
  scol.alloc(nnz > 0 ? nnz : 1, s);
  sval.alloc(nnz > 0 ? nnz : 1, s);
  k_sweep_fill<<<nb, 256, 0, s>>>(n, sch.order.get(), A.ptr.get(), A.col.get(), A.val.get(),
                                  forward ? 1 : 0, owner, full ? 1 : 0, sptr.get(), scol.get(), sval.get());
  MGRX_LAUNCH_CK();
  count_launch();
}

}  // namespace

// Diagnostic sweep trace (MGRX_GS_TRACE=<dir>): the first sweep of each
// schedule is run with %globaltimer stamps and written out with its order
// and dependency CSR for offline critical-path analysis.
struct Trace {
  DVec<unsigned long long> t0, t1;
  bool on = false;
};
void trace_begin(Trace& tr, const GsSchedule& sch, int n, cudaStream_t s) {
  static std::vector<const void*> seen;
  for (const void* k : seen)
    if (k == static_cast<const void*>(&sch)) return;
  seen.push_back(&sch);
  tr.on = true;
  tr.t0.alloc(n, s);
  tr.t1.alloc(n, s);
  unsigned long long* p0 = tr.t0.get();
  unsigned long long* p1 = tr.t1.get();
  MGRX_CK(cudaMemcpyToSymbolAsync(g_trace_start, &p0, sizeof(p0), 0, cudaMemcpyHostToDevice, s));
  MGRX_CK(cudaMemcpyToSymbolAsync(g_trace_pub, &p1, sizeof(p1), 0, cudaMemcpyHostToDevice, s));
}
void trace_end(Trace& tr, const char* dir, const GsSchedule& sch, int n, cudaStream_t s) {
  if (!tr.on) return;
  std::vector<unsigned long long> a = tr.t0.download(n), b = tr.t1.download(n);
  std::vector<int> ord = sch.order.download(n), dp = sch.dptr.download(n + 1);
  std::vector<int> dc = sch.dcol.download(dp[n] > 0 ? dp[n] : 1);
  unsigned long long* nul = nullptr;
  MGRX_CK(cudaMemcpyToSymbolAsync(g_trace_start, &nul, sizeof(nul), 0, cudaMemcpyHostToDevice, s));
  MGRX_CK(cudaMemcpyToSymbolAsync(g_trace_pub, &nul, sizeof(nul), 0, cudaMemcpyHostToDevice, s));
  MGRX_CK(cudaStreamSynchronize(s));
  char path[512];
  std::snprintf(path, sizeof path, "%s/gs_n%d_lv%d_%p.bin", dir, n, sch.levels, static_cast<const void*>(&sch));
  if (FILE* f = std::fopen(path, "wb")) {
    int hdr[3] = {n, sch.levels, dp[n]};
    std::fwrite(hdr, sizeof(int), 3, f);
    std::fwrite(ord.data(), sizeof(int), n, f);
    std::fwrite(dp.data(), sizeof(int), n + 1, f);
    std::fwrite(dc.data(), sizeof(int), dp[n], f);
    std::fwrite(a.data(), sizeof(unsigned long long), n, f);
    std::fwrite(b.data(), sizeof(unsigned long long), n, f);
    std::fclose(f);
  }
}

int gs_blk_rows() {
  static const int v = [] {
    const char* e = std::getenv("MGRX_GS_BLK_ROWS");
    const int r = e ? std::atoi(e) : kSmallN;
    return r <= 0 ? 0 : std::min(r, kSmallN);
  }();
  return v;
}

// Block plan of the block-partitioned sweep (see k_gs_blk and GsSchedule).
bool build_block_plan(const DCsr& A, bool forward, const double* d, const int* owner, GsSchedule& out,
                      cudaStream_t s) {
  const int n = A.rows;
  const int B = gs_blk_rows();
  if (B <= 0 || n <= B) return false;
  const HostCsr h = to_host(A, s);
  std::vector<int> own;
  if (owner) {
    own.resize(n);
    MGRX_CK(cudaMemcpyAsync(own.data(), owner, sizeof(int) * n, cudaMemcpyDeviceToHost, s));
  }
  std::vector<double> dh(n);
  MGRX_CK(cudaMemcpyAsync(dh.data(), d, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
  MGRX_CK(cudaStreamSynchronize(s));
  auto dep = [&](int i, int j) {
    return (forward ? j < i : j > i) && (own.empty() || own[j] == own[i]);
  };
  const int nb = (n + B - 1) / B;
  // MGRX_GS_BLK_ORDER=local: rows of a block by their block-local level
  // (intra-block dependencies only); default: by their global dependency
  // level, so every block walks the levels in the sweep's global order and
  // a block never waits on a later step of an earlier block
  static const bool local_order = [] {
    const char* e = std::getenv("MGRX_GS_BLK_ORDER");
    return e && e[0] == 'l';
  }();
  std::vector<int> glev;
  if (!local_order) {
    glev.assign(n, 0);
    for (int u = 0; u < n; ++u) {
      const int i = forward ? u : n - 1 - u;
      int m = 0;
      for (int k = h.ptr[i]; k < h.ptr[i + 1]; ++k) {
        const int j = h.col[k];
        if (dep(i, j)) m = std::max(m, glev[j] + 1);
      }
      glev[i] = m;
    }
  }
  std::vector<int> lev(n, 0);
  std::vector<int> pos_row, sp{0}, sc;
  std::vector<double> sv, sdv;
  std::vector<int> steps{0}, step_e, chunks{0}, blo, bch;
  step_e.push_back(0);
  for (int t = 0; t < nb; ++t) {
    const int b = forward ? t : nb - 1 - t;
    const int lo = b * B, hi = std::min(n, lo + B);
    int maxl = 0;
    for (int u = 0; u < hi - lo; ++u) {
      const int i = forward ? lo + u : hi - 1 - u;
      int m = 0;
      if (!local_order) {
        m = glev[i];
      } else {
        for (int k = h.ptr[i]; k < h.ptr[i + 1]; ++k) {
          const int j = h.col[k];
          if (dep(i, j) && j >= lo && j < hi) m = std::max(m, lev[j] + 1);
        }
      }
      lev[i] = m;
      maxl = std::max(maxl, m);
    }
    // rows by (local level, row index)
    std::vector<int> cnt(maxl + 2, 0);
    for (int i = lo; i < hi; ++i) ++cnt[lev[i] + 1];
    for (int l = 0; l <= maxl; ++l) cnt[l + 1] += cnt[l];
    std::vector<int> rows(hi - lo);
    {
      std::vector<int> at(cnt.begin(), cnt.end() - 1);
      for (int i = lo; i < hi; ++i) rows[at[lev[i]]++] = i;
    }
    blo.push_back(lo);
    bch.push_back(static_cast<int>(chunks.size()) - 1);
    const int pbase = static_cast<int>(pos_row.size());
    for (int i : rows) {
      pos_row.push_back(i);
      sdv.push_back(dh[i]);
      for (int k = h.ptr[i]; k < h.ptr[i + 1]; ++k) {
        const int j = h.col[k];
        if (!dep(i, j)) continue;
        sc.push_back((j >= lo && j < hi) ? j - lo : (j | kCrossBit));
        sv.push_back(h.val[k]);
      }
      if (static_cast<int>(sc.size()) - sp.back() > kSmallEnt) return false;
      sp.push_back(static_cast<int>(sc.size()));
    }
    // steps: runs of one local level within the buffer caps; chunks: runs
    // of consecutive steps within the same caps
    const int first_step = static_cast<int>(steps.size()) - 1;
    for (int l = 0; l <= maxl; ++l) {
      int p = pbase + cnt[l];
      const int pe = pbase + cnt[l + 1];
      while (p < pe) {
        int q = p;
        while (q < pe && q - p < kSmallRows && sp[q + 1] - sp[p] <= kSmallEnt) ++q;
        if (q == p) ++q;
        steps.push_back(q);
        step_e.push_back(sp[q]);
        p = q;
      }
    }
    const int last_step = static_cast<int>(steps.size()) - 1;
    int a = first_step;
    while (a < last_step) {
      int c = a + 1;
      while (c < last_step && steps[c + 1] - steps[a] <= kSmallRows && sp[steps[c + 1]] - sp[steps[a]] <= kSmallEnt)
        ++c;
      chunks.push_back(c);
      a = c;
    }
  }
  bch.push_back(static_cast<int>(chunks.size()) - 1);
  out.nblk = nb;
  out.blk_lo.alloc(nb, s);
  out.blk_lo.upload(blo.data(), nb);
  out.blk_chunk.alloc(nb + 1, s);
  out.blk_chunk.upload(bch.data(), nb + 1);
  out.border.alloc(n, s);
  out.border.upload(pos_row.data(), n);
  out.bsptr.alloc(n + 1, s);
  out.bsptr.upload(sp.data(), n + 1);
  const size_t ne = sc.size();
  out.bscol.alloc(ne > 0 ? ne : 1, s);
  out.bscol.upload(sc.data(), ne);
  out.bsval.alloc(ne > 0 ? ne : 1, s);
  out.bsval.upload(sv.data(), ne);
  out.bsd.alloc(n, s);
  out.bsd.upload(sdv.data(), n);
  out.bbp.alloc(n, s);
  out.nbsteps = static_cast<int>(steps.size()) - 1;
  std::vector<int> stv(steps);
  stv.insert(stv.end(), step_e.begin(), step_e.end());
  out.bsteps.alloc(stv.size(), s);
  out.bsteps.upload(stv.data(), stv.size());
  out.nbchunks = static_cast<int>(chunks.size()) - 1;
  out.bchunks.alloc(chunks.size(), s);
  out.bchunks.upload(chunks.data(), chunks.size());
  MGRX_CK(cudaStreamSynchronize(s));
  if (const char* v = std::getenv("MGRX_VERBOSE"); v && v[0] == '1') {
    int maxdepth = 0;
    for (int i = 0; i < n; ++i) maxdepth = std::max(maxdepth, lev[i] + 1);
    std::fprintf(stderr, "[mgrx] gs block plan: n=%d blocks=%d rows/block<=%d max local depth %d steps %d chunks %d\n",
                 n, nb, B, maxdepth, out.nbsteps, out.nbchunks);
  }
  return true;
}

void gs_schedule(const DCsr& A, bool forward, const double* d, bool full, GsSchedule& out,
                 cudaStream_t s, const int* owner) {
  const int n = A.rows;
  out.order.alloc(n > 0 ? n : 1, s);
  out.levels = 0;
  out.level_ptr.assign(1, 0);
  if (n == 0) return;
  DVec<int> lev(n, s), flag(1, s);
  lev.zero();
  const int nb = blocks_for(n, 256);
  while (true) {
    flag.zero();
    for (int it = 0; it < 8; ++it)
      k_levels<<<nb, 256, 0, s>>>(n, A.ptr.get(), A.col.get(), forward ? 1 : 0, owner, lev.get(),
                                  flag.get());
    MGRX_LAUNCH_CK();
    count_launch(8);
    if (read_scalar(flag.get(), s) == 0) break;
  }
  DVec<int> idx(n, s), lev_sorted(n, s);
  k_iota<<<nb, 256, 0, s>>>(n, idx.get());
  MGRX_LAUNCH_CK();
  count_launch();
  size_t tmp = 0;
  MGRX_CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, lev.get(), lev_sorted.get(), idx.get(),
                                          out.order.get(), n, 0, 31, s));
  DVec<char> t(tmp, s);
  MGRX_CK(cub::DeviceRadixSort::SortPairs(t.get(), tmp, lev.get(), lev_sorted.get(), idx.get(),
                                          out.order.get(), n, 0, 31, s));
  count_launch(4);
  const std::vector<int> ls = lev_sorted.download(n);
  out.levels = ls.back() + 1;
  out.level_ptr.assign(out.levels + 1, 0);
  for (int p = 0; p < n; ++p) ++out.level_ptr[ls[p] + 1];
  for (int l = 0; l < out.levels; ++l) out.level_ptr[l + 1] += out.level_ptr[l];

  build_sweep_csr(A, out, forward, owner, false, out.dptr, out.dcol, out.dval, s);
  out.has_full = full;
  if (full) build_sweep_csr(A, out, forward, owner, true, out.fptr, out.fcol, out.fval, s);
  out.sd.alloc(n, s);
  gather(n, out.order.get(), d, out.sd.get(), s);
  int dep_nnz = 0;
  MGRX_CK(cudaMemcpyAsync(&dep_nnz, out.dptr.get() + n, sizeof(int), cudaMemcpyDeviceToHost, s));
  MGRX_CK(cudaStreamSynchronize(s));
  const double avg = full ? (2.0 * dep_nnz) / n : static_cast<double>(dep_nnz) / n;
  out.team = avg <= 6.0 ? 1 : (avg <= 24.0 ? 4 : 8);
  out.dlptr.alloc(out.levels + 1, s);
  out.dlptr.upload(out.level_ptr.data(), out.levels + 1);
  // Sweep mode: MGRX_GS_MODE=lv selects the level-synchronous cluster
  // kernel; default is the sync-free kernel. Cluster size from the
  // average level width (about 1 row per thread).
  // 0 sync-free (default, fastest measured at cfg2: 2-3 us per dependency
  // hop), 1 level-synchronous cluster (MGRX_GS_MODE=lv), 2 pipelined single
  // CTA (MGRX_GS_MODE=pipe); both alternatives measured 2-4x slower.
  static const int mode = [] {
    const char* e = std::getenv("MGRX_GS_MODE");
    if (e && e[0] == 'l') return 1;
    if (e && e[0] == 'p') return 2;
    return 0;
  }();
  if (mode == 1) {
    const double width = static_cast<double>(n) / out.levels;
    out.cluster = std::max(1, std::min(16, static_cast<int>(std::ceil(width / kLvThreads))));
  } else {
    out.cluster = 0;
  }
  out.pipe = 0;
  out.small = 0;
  if (n <= kSmallN && mode == 0) {
    const std::vector<int> dp = out.dptr.download(n + 1);
    bool ok = true;
    for (int q = 0; q < n && ok; ++q) ok = dp[q + 1] - dp[q] <= kSmallEnt;
    std::vector<int> fp;
    if (ok && full) {
      fp = out.fptr.download(n + 1);
      for (int q = 0; q < n && ok; ++q) ok = fp[q + 1] - fp[q] <= kSmallEnt;
    }
    if (ok) {
      auto with_offsets = [](const std::vector<int>& st, const std::vector<int>& ptr) {
        std::vector<int> v(st);
        for (int q : st) v.push_back(ptr[q]);
        return v;
      };
      const std::vector<int> st = pipe_steps(out.level_ptr, dp, kSmallRows, kSmallEnt);
      out.ndsteps = static_cast<int>(st.size()) - 1;
      const std::vector<int> stv = with_offsets(st, dp);
      out.dsteps.alloc(stv.size(), s);
      out.dsteps.upload(stv.data(), stv.size());
      const std::vector<int> ch = small_chunks(st, dp, kSmallRows, kSmallEnt);
      out.ndchunks = static_cast<int>(ch.size()) - 1;
      out.dchunks.alloc(ch.size(), s);
      out.dchunks.upload(ch.data(), ch.size());
      if (full) {
        const std::vector<int> st2 = pipe_steps(out.level_ptr, fp, kSmallRows, kSmallEnt);
        out.nfsteps = static_cast<int>(st2.size()) - 1;
        const std::vector<int> stv2 = with_offsets(st2, fp);
        out.fsteps.alloc(stv2.size(), s);
        out.fsteps.upload(stv2.data(), stv2.size());
        const std::vector<int> ch2 = small_chunks(st2, fp, kSmallRows, kSmallEnt);
        out.nfchunks = static_cast<int>(ch2.size()) - 1;
        out.fchunks.alloc(ch2.size(), s);
        out.fchunks.upload(ch2.data(), ch2.size());
      }
      out.bp.alloc(n, s);
      out.small = 1;
    }
  }
  out.blk = 0;
  if (n > kSmallN && mode == 0 && !out.small && build_block_plan(A, forward, d, owner, out, s)) {
    // keep the block-partitioned sweep only where it times faster than the
    // sync-free one (it wins on structured levels whose row blocks carry
    // their dependency chains, loses on coarse levels whose blocks couple at
    // every dependency level): best of two timed sweeps each, from zero
    GsScratch scr;
    gs_bind_scratch(scr, s);
    DVec<double> bb(n, s), xx(n, s);
    std::vector<double> ones(n, 1.0);
    bb.upload(ones.data(), n);
    cudaEvent_t e0, e1;
    MGRX_CK(cudaEventCreate(&e0));
    MGRX_CK(cudaEventCreate(&e1));
    auto time_mode = [&](int blk) {
      out.blk = blk;
      float best = 1e30f;
      for (int r = 0; r < 3; ++r) {
        MGRX_CK(cudaEventRecord(e0, s));
        gs_sweep(A, out, d, bb.get(), nullptr, xx.get(), nullptr, forward, scr, s);
        MGRX_CK(cudaEventRecord(e1, s));
        MGRX_CK(cudaEventSynchronize(e1));
        float ms = 0.0f;
        MGRX_CK(cudaEventElapsedTime(&ms, e0, e1));
        if (r > 0) best = std::min(best, ms);
      }
      return best;
    };
    const float tb = time_mode(1), tf = time_mode(0);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    gs_check(scr, s);
    out.blk = tb < tf ? 1 : 0;
    if (const char* v = std::getenv("MGRX_VERBOSE"); v && v[0] == '1')
      std::fprintf(stderr, "[mgrx] gs sweep n=%d: block %.1f us, sync-free %.1f us -> %s\n", n, tb * 1e3, tf * 1e3,
                   out.blk ? "block" : "sync-free");
    if (std::getenv("MGRX_GS_BLK_FORCE")) out.blk = 1;
  }
  if (mode == 2) {
    const std::vector<int> dp = out.dptr.download(n + 1);
    bool ok = true;
    for (int q = 0; q < n && ok; ++q) ok = dp[q + 1] - dp[q] <= kPipeEnt;
    std::vector<int> fp;
    if (ok && full) {
      fp = out.fptr.download(n + 1);
      for (int q = 0; q < n && ok; ++q) ok = fp[q + 1] - fp[q] <= kPipeEnt;
    }
    if (ok) {
      auto with_offsets = [](const std::vector<int>& st, const std::vector<int>& ptr) {
        std::vector<int> v(st);
        for (int q : st) v.push_back(ptr[q]);
        return v;
      };
      const std::vector<int> st = pipe_steps(out.level_ptr, dp);
      out.ndsteps = static_cast<int>(st.size()) - 1;
      const std::vector<int> stv = with_offsets(st, dp);
      out.dsteps.alloc(stv.size(), s);
      out.dsteps.upload(stv.data(), stv.size());
      if (full) {
        const std::vector<int> st2 = pipe_steps(out.level_ptr, fp);
        out.nfsteps = static_cast<int>(st2.size()) - 1;
        const std::vector<int> stv2 = with_offsets(st2, fp);
        out.fsteps.alloc(stv2.size(), s);
        out.fsteps.upload(stv2.data(), stv2.size());
      }
      out.bp.alloc(n, s);
      out.pipe = 1;
    }
  }
}

void gs_sweep(const DCsr& A, const GsSchedule& sch, const double* d, const double* b,
              const double* xold, double* xnew, double* zadd, bool forward, GsScratch& scr,
              cudaStream_t s) {
  (void)d;
  (void)forward;
  const int n = A.rows;
  if (n == 0) return;
  if (scr.ticket_err.size() < 2) throw RuntimeError("gs_sweep: scratch not bound");
  const bool full_sweep = xold != nullptr;
  if (full_sweep && !sch.has_full) throw RuntimeError("gs_sweep: schedule built without the full sweep CSR");
  if (sch.small) {
    k_gather_d<<<blocks_for(n, 256), 256, 0, s>>>(n, sch.order.get(), b, const_cast<double*>(sch.bp.get()));
    const int* sp = full_sweep ? sch.fptr.get() : sch.dptr.get();
    const int* sc = full_sweep ? sch.fcol.get() : sch.dcol.get();
    const double* sv = full_sweep ? sch.fval.get() : sch.dval.get();
    if (full_sweep)
      k_gs_small<true><<<1, kPipeThreads, kSmallSmem, s>>>(sch.nfsteps, sch.fsteps.get(), sch.nfchunks,
                                                           sch.fchunks.get(), sch.order.get(), sp, sc, sv,
                                                           sch.sd.get(), sch.bp.get(), xold, xnew, zadd);
    else
      k_gs_small<false><<<1, kPipeThreads, kSmallSmem, s>>>(sch.ndsteps, sch.dsteps.get(), sch.ndchunks,
                                                            sch.dchunks.get(), sch.order.get(), sp, sc, sv,
                                                            sch.sd.get(), sch.bp.get(), xold, xnew, zadd);
    MGRX_LAUNCH_CK();
    count_launch(2);
    return;
  }
  if (sch.blk && !full_sweep) {
    MGRX_CK(cudaMemsetAsync(scr.ticket_err.get(), 0, sizeof(int), s));
    MGRX_CK(cudaMemsetAsync(xnew, 0xff, sizeof(double) * n, s));
    k_gather_d<<<blocks_for(n, 256), 256, 0, s>>>(n, sch.border.get(), b, const_cast<double*>(sch.bbp.get()));
    const int grid = std::min(sch.nblk, device_sms());
    k_gs_blk<<<grid, kPipeThreads, kSmallSmem, s>>>(sch.nblk, sch.blk_lo.get(), sch.blk_chunk.get(), sch.nbsteps,
                                                     sch.bsteps.get(), sch.bchunks.get(), sch.border.get(),
                                                     sch.bsptr.get(), sch.bscol.get(), sch.bsval.get(),
                                                     sch.bsd.get(), sch.bbp.get(), xnew, zadd, scr.ticket_err.get());
    MGRX_LAUNCH_CK();
    count_launch(2);
    return;
  }
  if (sch.pipe) {
    k_gather_d<<<blocks_for(n, 256), 256, 0, s>>>(n, sch.order.get(), b, const_cast<double*>(sch.bp.get()));
    const int* sp = full_sweep ? sch.fptr.get() : sch.dptr.get();
    const int* sc = full_sweep ? sch.fcol.get() : sch.dcol.get();
    const double* sv = full_sweep ? sch.fval.get() : sch.dval.get();
    if (full_sweep)
      k_gs_pipe<true><<<1, kPipeThreads, kPipeSmem, s>>>(sch.nfsteps, sch.fsteps.get(), sch.order.get(), sp, sc,
                                                         sv, sch.sd.get(), sch.bp.get(), xold, xnew, zadd);
    else
      k_gs_pipe<false><<<1, kPipeThreads, kPipeSmem, s>>>(sch.ndsteps, sch.dsteps.get(), sch.order.get(), sp, sc,
                                                          sv, sch.sd.get(), sch.bp.get(), xold, xnew, zadd);
    MGRX_LAUNCH_CK();
    count_launch(2);
    return;
  }
  if (sch.cluster > 0) {
    // level-synchronous cluster sweep
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sch.cluster);
    cfg.blockDim = dim3(kLvThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = sch.cluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const int* sp = full_sweep ? sch.fptr.get() : sch.dptr.get();
    const int* sc = full_sweep ? sch.fcol.get() : sch.dcol.get();
    const double* sv = full_sweep ? sch.fval.get() : sch.dval.get();
    const bool clus = sch.cluster > 1;
    if (!clus) cfg.numAttrs = 0;
    if (full_sweep && clus)
      MGRX_CK(cudaLaunchKernelEx(&cfg, k_gs_lv<true, true>, sch.levels, sch.dlptr.get(), sch.order.get(), sp,
                                 sc, sv, sch.sd.get(), b, xold, xnew, zadd));
    else if (full_sweep)
      MGRX_CK(cudaLaunchKernelEx(&cfg, k_gs_lv<true, false>, sch.levels, sch.dlptr.get(), sch.order.get(), sp,
                                 sc, sv, sch.sd.get(), b, xold, xnew, zadd));
    else if (clus)
      MGRX_CK(cudaLaunchKernelEx(&cfg, k_gs_lv<false, true>, sch.levels, sch.dlptr.get(), sch.order.get(), sp,
                                 sc, sv, sch.sd.get(), b, xold, xnew, zadd));
    else
      MGRX_CK(cudaLaunchKernelEx(&cfg, k_gs_lv<false, false>, sch.levels, sch.dlptr.get(), sch.order.get(), sp,
                                 sc, sv, sch.sd.get(), b, xold, xnew, zadd));
    count_launch();
    return;
  }
  MGRX_CK(cudaMemsetAsync(scr.ticket_err.get(), 0, sizeof(int), s));
  MGRX_CK(cudaMemsetAsync(xnew, 0xff, sizeof(double) * n, s));
  // Team size from the average dependency count; grid: enough CTAs to keep
  // ~kFlight dependency levels of rows in flight.
  static const int kFlight = [] {
    const char* e = std::getenv("MGRX_GS_FLIGHT");
    return e ? std::max(1, std::atoi(e)) : 6;
  }();
  const bool full = full_sweep;
  const int T = sch.team;
  const double per_level = static_cast<double>(n) / std::max(sch.levels, 1);
  const int rows_per_cta = kGsThreads / T;
  const int grid = std::max(1, std::min(blocks_for(n, rows_per_cta),
                                        static_cast<int>(kFlight * per_level / rows_per_cta) + 1));
  const int* sp = full ? sch.fptr.get() : sch.dptr.get();
  const int* sc = full ? sch.fcol.get() : sch.dcol.get();
  const double* sv = full ? sch.fval.get() : sch.dval.get();
  int* tk = scr.ticket_err.get();
  static const unsigned kSleep = [] {
    const char* e = std::getenv("MGRX_GS_SLEEP");
    return e ? static_cast<unsigned>(std::atoi(e)) : 20u;
  }();
  static const int kPub = [] {
    const char* e = std::getenv("MGRX_GS_PUB");
    return e ? std::atoi(e) : 0;
  }();
  const char* trace_dir = std::getenv("MGRX_GS_TRACE");
  Trace tr;
  if (trace_dir && !full) trace_begin(tr, sch, n, s);
#define MGRX_GS_LAUNCH(TT, FF)                                                                    \
  k_gs<TT, FF><<<grid, kGsThreads, kGsSmem, s>>>(n, sch.order.get(), sp, sc, sv, sch.sd.get(), b, \
                                                 xold, xnew, zadd, tk, kSleep, kPub)
  if (T == 1) {
    if (full) MGRX_GS_LAUNCH(1, true); else MGRX_GS_LAUNCH(1, false);
  } else if (T == 4) {
    if (full) MGRX_GS_LAUNCH(4, true); else MGRX_GS_LAUNCH(4, false);
  } else {
    if (full) MGRX_GS_LAUNCH(8, true); else MGRX_GS_LAUNCH(8, false);
  }
#undef MGRX_GS_LAUNCH
  if (trace_dir) trace_end(tr, trace_dir, sch, n, s);
  MGRX_LAUNCH_CK();
  count_launch();
}

void gs_bind_scratch(GsScratch& scr, cudaStream_t s) {
  if (first_on_device(reinterpret_cast<const void*>(&gs_bind_scratch))) {
    MGRX_CK(cudaFuncSetAttribute(k_gs_small<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmallSmem)));
    MGRX_CK(cudaFuncSetAttribute(k_gs_small<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmallSmem)));
    MGRX_CK(cudaFuncSetAttribute(k_gs_blk, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmallSmem)));
    MGRX_CK(cudaFuncSetAttribute(k_gs_pipe<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kPipeSmem)));
    MGRX_CK(cudaFuncSetAttribute(k_gs_pipe<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kPipeSmem)));
    MGRX_CK(cudaFuncSetAttribute(k_gs_lv<false, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    MGRX_CK(cudaFuncSetAttribute(k_gs_lv<true, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    const int sm = static_cast<int>(kGsSmem);
    MGRX_CK(cudaFuncSetAttribute(k_gs<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    MGRX_CK(cudaFuncSetAttribute(k_gs<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    MGRX_CK(cudaFuncSetAttribute(k_gs<4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    MGRX_CK(cudaFuncSetAttribute(k_gs<4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    MGRX_CK(cudaFuncSetAttribute(k_gs<8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    MGRX_CK(cudaFuncSetAttribute(k_gs<8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
  }
  if (scr.ticket_err.size() < 2) {
    scr.ticket_err.alloc(2, s);
    scr.ticket_err.zero();
  }
}

void gs_check(GsScratch& scr, cudaStream_t s) {
  if (scr.ticket_err.size() < 2) return;
  const int e = read_scalar(scr.ticket_err.get() + 1, s);
  if (e) throw RuntimeError("gauss-seidel sweep exceeded its dependency wait limit");
}

void jacobi0(int n, double w, const double* dinv, const double* r, const int* rrow, double* z,
             cudaStream_t s) {
  if (n == 0) return;
  launch_pdl(k_jacobi0, blocks_for(n, 512), 256, 0, s, n, w, dinv, r, rrow, z);
  MGRX_LAUNCH_CK();
  count_launch();
}

void vec_add(int n, const double* a, double* y, cudaStream_t s) {
  if (n == 0) return;
  launch_pdl(k_vec_add, blocks_for(n, 256), 256, 0, s, n, a, y);
  MGRX_LAUNCH_CK();
  count_launch();
}

void gather(int n, const int* idx, const double* x, double* y, cudaStream_t s) {
  if (n == 0) return;
  launch_pdl(k_gather, blocks_for(n, 256), 256, 0, s, n, idx, x, y);
  MGRX_LAUNCH_CK();
  count_launch();
}

void reciprocal(int n, const double* d, double* y, cudaStream_t s) {
  if (n == 0) return;
  k_recip<<<blocks_for(n, 256), 256, 0, s>>>(n, d, y);
  MGRX_LAUNCH_CK();
  count_launch();
}

}  // namespace mgrx
