// Smoother kernels. The Gauss-Seidel sweep is the reference's sequential
// loop (proj/src/relax.cpp:55-78, one range) executed sync-free: rows are
// dispatched in dependency-level order through a ticket counter, and each
// row polls the values it depends on. A value doubles as its own ready flag:
// xnew is pre-filled with an all-ones NaN pattern that no finite result can
// produce, and a finished row publishes its 64-bit result with one relaxed
// gpu-scope store. Every row performs exactly the reference's operations in
// the reference's order, so the result is bitwise equal to the CPU loop.
#include <cub/cub.cuh>

#include "relax.cuh"

namespace mgrx {
namespace {

constexpr int kGsThreads = 128;
constexpr long long kSpinLimit = 1LL << 24;

__device__ __forceinline__ double ld_relaxed(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ int ld_relaxed_int(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Each lane owns one row and walks it in register-resident chunks of kChunk
// entries: the chunk's columns/values (and the old values of non-dependency
// columns) are loaded up front, all pending dependencies are polled in
// parallel, and the chunk is folded into the row sum in stored order only
// once every value is present. A lane that finds a dependency still pending
// backs off briefly so spinning warps do not crowd out producing ones.
constexpr int kChunk = 16;

__global__ void __launch_bounds__(kGsThreads)
    k_gs(int n, const int* __restrict__ order, const int* __restrict__ ptr,
         const int* __restrict__ col, const double* __restrict__ val, const double* __restrict__ d,
         const double* __restrict__ b, const double* __restrict__ xold, double* xnew, double* zadd,
         int fwd, int* tk) {
  __shared__ int base;
  if (threadIdx.x == 0) base = atomicAdd(tk, kGsThreads);
  __syncthreads();
  const int pos = base + threadIdx.x;
  const bool active = pos < n;
  int i = 0, k = 0, ke = 0;
  double s = 0.0;
  if (active) {
    i = order[pos];
    k = ptr[i];
    ke = ptr[i + 1];
    s = b[i];
  }
  int cc[kChunk];
  double cv[kChunk], xv[kChunk];
  unsigned pending = 0;
  int cn = 0;
  auto load_chunk = [&]() {
    cn = min(kChunk, ke - k);
    pending = 0;
#pragma unroll
    for (int q = 0; q < kChunk; ++q) {
      if (q < cn) {
        cc[q] = col[k + q];
        cv[q] = val[k + q];
        const bool dep = fwd ? (cc[q] < i) : (cc[q] > i);
        if (dep) pending |= 1u << q;
        else xv[q] = xold ? xold[cc[q]] : 0.0;
      }
    }
  };
  if (active) load_chunk();
  bool done = !active;
  long long spins = 0;
  while (!__all_sync(0xffffffffu, done)) {
    if (!done) {
#pragma unroll
      for (int q = 0; q < kChunk; ++q) {
        if (pending & (1u << q)) {
          const double v = ld_relaxed(xnew + cc[q]);
          if (__double_as_longlong(v) != -1LL) {
            xv[q] = v;
            pending &= ~(1u << q);
          }
        }
      }
      if (pending == 0) {
#pragma unroll
        for (int q = 0; q < kChunk; ++q)
          if (q < cn) s = __dsub_rn(s, __dmul_rn(cv[q], xv[q]));
        k += cn;
        if (k >= ke) {
          const double xi = xold ? xold[i] : 0.0;
          const double v = __dadd_rn(xi, __ddiv_rn(s, d[i]));
          st_relaxed(xnew + i, v);
          if (zadd) zadd[i] = __dadd_rn(zadd[i], v);
          done = true;
        } else {
          load_chunk();
        }
      } else if (++spins > kSpinLimit) {
        atomicExch(tk + 1, 1);
        st_relaxed(xnew + i, 0.0);
        done = true;
      } else {
        __nanosleep(32);
      }
    }
  }
}

// Dependency levels by monotone in-place relaxation: lev[i] = 1 + max over
// dependencies; converges to the longest-path level.
__global__ void k_levels(int n, const int* __restrict__ ptr, const int* __restrict__ col, int fwd,
                         int* lev, int* changed) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int m = 0;
  for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
    const int j = col[k];
    if (fwd ? (j < i) : (j > i)) {
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
__global__ void k_jacobi0(int n, double w, const double* __restrict__ dinv,
                          const double* __restrict__ r, const int* __restrict__ rrow,
                          double* __restrict__ z) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double rv = rrow ? r[rrow[i]] : r[i];
  z[i] = __dmul_rn(w, __dmul_rn(dinv[i], rv));
}
__global__ void k_vec_add(int n, const double* __restrict__ a, double* __restrict__ y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = __dadd_rn(y[i], a[i]);
}
__global__ void k_gather(int n, const int* __restrict__ idx, const double* __restrict__ x,
                         double* __restrict__ y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = x[idx[i]];
}

__global__ void k_recip(int n, const double* __restrict__ d, double* __restrict__ y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = __ddiv_rn(1.0, d[i]);
}

}  // namespace

void gs_schedule(const DCsr& A, bool forward, GsSchedule& out, cudaStream_t s) {
  const int n = A.rows;
  out.order.alloc(n > 0 ? n : 1, s);
  out.levels = 0;
  if (n == 0) return;
  DVec<int> lev(n, s), flag(1, s);
  lev.zero();
  const int nb = blocks_for(n, 256);
  while (true) {
    flag.zero();
    for (int it = 0; it < 8; ++it)
      k_levels<<<nb, 256, 0, s>>>(n, A.ptr.get(), A.col.get(), forward ? 1 : 0, lev.get(), flag.get());
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
  out.levels = read_scalar(lev_sorted.get() + (n - 1), s) + 1;
}

void gs_sweep(const DCsr& A, const GsSchedule& sch, const double* d, const double* b,
              const double* xold, double* xnew, double* zadd, bool forward, GsScratch& scr,
              cudaStream_t s) {
  const int n = A.rows;
  if (n == 0) return;
  if (scr.ticket_err.size() < 2) throw RuntimeError("gs_sweep: scratch not bound");
  MGRX_CK(cudaMemsetAsync(scr.ticket_err.get(), 0, sizeof(int), s));
  MGRX_CK(cudaMemsetAsync(xnew, 0xff, sizeof(double) * n, s));
  k_gs<<<blocks_for(n, kGsThreads), kGsThreads, 0, s>>>(n, sch.order.get(), A.ptr.get(), A.col.get(),
                                                       A.val.get(), d, b, xold, xnew, zadd,
                                                       forward ? 1 : 0, scr.ticket_err.get());
  MGRX_LAUNCH_CK();
  count_launch();
}

void gs_bind_scratch(GsScratch& scr, cudaStream_t s) {
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
  k_jacobi0<<<blocks_for(n, 256), 256, 0, s>>>(n, w, dinv, r, rrow, z);
  MGRX_LAUNCH_CK();
  count_launch();
}

void vec_add(int n, const double* a, double* y, cudaStream_t s) {
  if (n == 0) return;
  k_vec_add<<<blocks_for(n, 256), 256, 0, s>>>(n, a, y);
  MGRX_LAUNCH_CK();
  count_launch();
}

void gather(int n, const int* idx, const double* x, double* y, cudaStream_t s) {
  if (n == 0) return;
  k_gather<<<blocks_for(n, 256), 256, 0, s>>>(n, idx, x, y);
  MGRX_LAUNCH_CK();
  count_launch();
}

}  // namespace mgrx

namespace mgrx {
void reciprocal(int n, const double* d, double* y, cudaStream_t s) {
  if (n == 0) return;
  k_recip<<<blocks_for(n, 256), 256, 0, s>>>(n, d, y);
  MGRX_LAUNCH_CK();
  count_launch();
}
}  // namespace mgrx
