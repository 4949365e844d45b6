// Device GMRES. Each modified Gram-Schmidt step is one fused kernel: it
// applies the previous projection (w -= h_{i-1} v_{i-1}, with h read from HBM
// so nothing waits on the host) and reduces the next inner product v_i . w in
// the same pass. Reductions use a fixed grid and a fixed tree, with the last
// CTA folding the per-CTA partials in index order, so every run is bitwise
// reproducible. The host reads the Hessenberg column once per step (one
// small D2H copy), exactly where the reference needs scalar control flow.
#include <cmath>

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

// w <- w - (*hprev) * vprev (if vprev); then dot1 = sum a_i w_i (if a),
// dot2 = sum w_i w_i (if want2). Results: out1 (and hacc = / += dot1), out2.
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
  int i0 = blockIdx.x * kRT + threadIdx.x;
  for (; i0 + (kU - 1) * kStride < n; i0 += kU * kStride) {
    double wv[kU], pv[kU], av[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = i0 + u * kStride;
      wv[u] = __ldcg(w + i);
      if (vprev) pv[u] = __ldcg(vprev + i);
      if (a) av[u] = __ldcg(a + i);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      double wi = wv[u];
      if (vprev) {
        wi = __dsub_rn(wi, __dmul_rn(h, pv[u]));
        w[i0 + u * kStride] = wi;
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
  k_mgs<<<kRB, kRT, 0, s>>>(n, w, vprev, hprev, a, want2 ? 1 : 0, ws.part.get(), ws.ctr.get(), out1,
                            hacc, accumulate ? 1 : 0, out2);
  MGRX_LAUNCH_CK();
  count_launch();
}

}  // namespace

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

double device_dot(int n, const double* a, const double* b, GmresWork& ws, cudaStream_t s) {
  // dot(a, b) = sum a_i b_i via the MGS kernel with w = b, no projection.
  mgs_launch(n, const_cast<double*>(b), nullptr, nullptr, a, false, ws, ws.scal.get(), nullptr,
             false, nullptr, s);
  return read_scalar(ws.scal.get(), s);
}

GmresResult gmres_device(const DCsr& A, const double* b, double* x, const KrylovSpec& cfg,
                         const DevOp& precond, GmresWork& ws, cudaStream_t s) {
  const int n = A.rows;
  if (cfg.restart < 1) throw InvalidArgument("gmres: restart must be >= 1");
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
        prec(col(k), ws.z.get());
        spmv(A, ws.z.get(), ws.w.get(), s);  // w = A M^{-1} v_k
        // pass 1: h_i = v_i . w ; w -= h_i v_i  (krylov.cpp:84-89)
        for (int i = 0; i <= k; ++i)
          mgs_launch(n, ws.w.get(), i ? col(i - 1) : nullptr, i ? s_hp + (i - 1) : nullptr, col(i),
                     i == 0, ws, s_hp + i, s_hc + i, false, i == 0 ? s_n0 : nullptr, s);
        mgs_launch(n, ws.w.get(), col(k), s_hp + k, nullptr, true, ws, nullptr, nullptr, false, s_n1, s);
        MGRX_CK(cudaMemcpyAsync(H_pin, S, col_bytes, cudaMemcpyDeviceToHost, s));
        MGRX_CK(cudaStreamSynchronize(s));
        const double w0 = std::sqrt(H_pin[0]);
        double wn = std::sqrt(H_pin[1]);
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
        const double* hc = H_pin + 3 + (m + 1);
        for (int i = 0; i <= k; ++i) h(i, k) = hc[i];
        h(k + 1, k) = wn;
        if (!std::isfinite(wn)) throw RuntimeError("gmres: Arnoldi vector is non-finite");
        const bool happy = wn < 1e-300;
        if (!happy) {
          k_scale<<<blocks_for(n, 256), 256, 0, s>>>(n, ws.w.get(), wn, col(k + 1));
          MGRX_LAUNCH_CK();
          count_launch();
        }
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
