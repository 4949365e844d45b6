// Single-CTA AMG tail (see amgtail.cuh). One CTA of kTT threads holds the
// tail's operators and work vectors in shared memory and runs
//   down:  z_l = S_pre(r_l); t_l = r_l - A_l z_l; r_{l+1} = R_l t_l
//   coarsest: z_c = LU \ r_c
//   up:    z_l += P_l z_{l+1}; t_l = r_l - A_l z_l; z_l += S_post(t_l)
// with the operation-for-operation arithmetic of the launch-per-operation
// path: SpMV rows summed left to right from 0.0 (EpiStore adds 0.0, the
// residual forms b - (0 + s), the prolongation y + s), Jacobi sweeps as
// spmv_jacobi_ex (the zero-start iterate w*(dinv*b), later sweeps
// z + w*(dinv*(b - (0 + s)))), post-smoothing accumulated with z + v, the
// dense solve as DenseLU's (x_i -= l_ij x_j for j ascending, then x_j /= u_jj
// before x_i -= u_ij x_j for j descending).
#include <algorithm>
#include <cstring>

#include "amgtail.cuh"

namespace mgrx {
namespace {

constexpr int kTT = 512;

template <class T>
__device__ __forceinline__ T* at(unsigned char* base, int off) {
  return reinterpret_cast<T*>(base + off);
}

// y_i = epi(i, sum_k val_k x_col_k) over rows i < m (thread per row)
template <class Epi>
__device__ __forceinline__ void tail_spmv(int m, const int* ptr, const int* col, const double* val, const double* x,
                                          Epi epi) {
  for (int i = threadIdx.x; i < m; i += kTT) {
    double s = 0.0;
    for (int k = ptr[i]; k < ptr[i + 1]; ++k) s = __dadd_rn(s, __dmul_rn(val[k], x[col[k]]));
    epi(i, s);
  }
}

// z = S(b) (acc == false) or z += S(b) (acc == true), S = `sweeps` weighted
// Jacobi sweeps from zero with inverse diagonal dinv. v1, v2: scratch.
__device__ void tail_jacobi(int m, const int* ptr, const int* col, const double* val, const double* dinv, double w,
                            int sweeps, const double* b, double* z, bool acc, double* v1, double* v2) {
  if (sweeps <= 1) {
    for (int i = threadIdx.x; i < m; i += kTT) {
      const double v = __dmul_rn(w, __dmul_rn(dinv[i], b[i]));
      z[i] = acc ? __dadd_rn(z[i], v) : v;
    }
    __syncthreads();
    return;
  }
  for (int i = threadIdx.x; i < m; i += kTT) v1[i] = __dmul_rn(w, __dmul_rn(dinv[i], b[i]));
  __syncthreads();
  const double* cur = v1;
  for (int sw = 1; sw < sweeps; ++sw) {
    const bool last = sw == sweeps - 1;
    double* nxt = last ? z : (cur == v1 ? v2 : v1);
    tail_spmv(m, ptr, col, val, cur, [&](int i, double s) {
      const double d = __dsub_rn(b[i], __dadd_rn(0.0, s));
      const double v = __dadd_rn(cur[i], __dmul_rn(w, __dmul_rn(dinv[i], d)));
      nxt[i] = (last && acc) ? __dadd_rn(z[i], v) : v;
    });
    __syncthreads();
    cur = nxt;
  }
}

__global__ void __launch_bounds__(kTT, 1) k_amg_tail(TailDesc d, const unsigned char* __restrict__ blob,
                                                    const double* __restrict__ r, double* __restrict__ z) {
  pdl_enter();
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ __align__(8) unsigned long long mbar;
  const int T = threadIdx.x;
  const unsigned mb = static_cast<unsigned>(__cvta_generic_to_shared(&mbar));
  if (T == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(mb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(mb), "r"(d.blob_bytes) : "memory");
    constexpr int kChunk = 32768;
    for (int o = 0; o < d.blob_bytes; o += kChunk) {
      const int nb = min(kChunk, d.blob_bytes - o);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              static_cast<unsigned>(__cvta_generic_to_shared(sm + o))),
          "l"(blob + o), "r"(nb), "r"(mb)
          : "memory");
    }
  }
  {
    double* r0 = at<double>(sm, d.L[0].vr);
    for (int i = T; i < d.L[0].m; i += kTT) r0[i] = r[i];
  }
  __syncthreads();  // mbarrier initialised before anyone waits on it
  unsigned done = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done)
                 : "r"(mb), "r"(0u)
                 : "memory");
  } while (!done);
  __syncthreads();

  // down
  for (int l = 0; l < d.nlev; ++l) {
    const TailLevel& L = d.L[l];
    const int* ap = at<int>(sm, L.a_ptr);
    const int* ac = at<int>(sm, L.a_col);
    const double* av = at<double>(sm, L.a_val);
    double* rl = at<double>(sm, L.vr);
    double* zl = at<double>(sm, L.vz);
    double* tl = at<double>(sm, L.vt);
    tail_jacobi(L.m, ap, ac, av, at<double>(sm, L.dpre), L.pre_w, L.pre_sweeps, rl, zl, false, at<double>(sm, L.v1),
                at<double>(sm, L.v2));
    tail_spmv(L.m, ap, ac, av, zl, [&](int i, double s) { tl[i] = __dsub_rn(rl[i], __dadd_rn(0.0, s)); });
    __syncthreads();
    double* rn = at<double>(sm, l + 1 < d.nlev ? d.L[l + 1].vr : d.cr);
    tail_spmv(L.mc, at<int>(sm, L.r_ptr), at<int>(sm, L.r_col), at<double>(sm, L.r_val), tl,
              [&](int i, double s) { rn[i] = __dadd_rn(0.0, s); });
    __syncthreads();
  }
  // coarsest: one warp, column sweeps in the dense algorithm's order
  if (T < 32) {
    const int n = d.nc;
    const double* M = at<double>(sm, d.lu);
    const int* pm = at<int>(sm, d.perm);
    const double* rc = at<double>(sm, d.cr);
    double* xs = at<double>(sm, d.cz);
    for (int i = T; i < n; i += 32) xs[i] = rc[pm[i]];
    __syncwarp();
    for (int j = 0; j < n; ++j) {
      const double xj = xs[j];
      for (int i = j + 1 + T; i < n; i += 32) xs[i] = __dsub_rn(xs[i], __dmul_rn(M[static_cast<size_t>(j) * n + i], xj));
      __syncwarp();
    }
    for (int j = n - 1; j >= 0; --j) {
      if (T == 0) xs[j] = __ddiv_rn(xs[j], M[static_cast<size_t>(j) * n + j]);
      __syncwarp();
      const double xj = xs[j];
      for (int i = T; i < j; i += 32) xs[i] = __dsub_rn(xs[i], __dmul_rn(M[static_cast<size_t>(j) * n + i], xj));
      __syncwarp();
    }
  }
  __syncthreads();
  // up
  for (int l = d.nlev - 1; l >= 0; --l) {
    const TailLevel& L = d.L[l];
    const int* ap = at<int>(sm, L.a_ptr);
    const int* ac = at<int>(sm, L.a_col);
    const double* av = at<double>(sm, L.a_val);
    double* rl = at<double>(sm, L.vr);
    double* zl = at<double>(sm, L.vz);
    double* tl = at<double>(sm, L.vt);
    const double* en = at<double>(sm, l + 1 < d.nlev ? d.L[l + 1].vz : d.cz);
    tail_spmv(L.m, at<int>(sm, L.p_ptr), at<int>(sm, L.p_col), at<double>(sm, L.p_val), en,
              [&](int i, double s) { zl[i] = __dadd_rn(zl[i], s); });
    __syncthreads();
    tail_spmv(L.m, ap, ac, av, zl, [&](int i, double s) { tl[i] = __dsub_rn(rl[i], __dadd_rn(0.0, s)); });
    __syncthreads();
    tail_jacobi(L.m, ap, ac, av, at<double>(sm, L.dpost), L.post_w, L.post_sweeps, tl, zl, true,
                at<double>(sm, L.v1), at<double>(sm, L.v2));
  }
  const double* z0 = at<double>(sm, d.L[0].vz);
  for (int i = T; i < d.L[0].m; i += kTT) z[i] = z0[i];
}

}  // namespace

bool build_tail_blob(const std::vector<TailLevelHost>& lv, int nc, const std::vector<double>& lu,
                     const std::vector<int>& perm, size_t max_bytes, TailDesc& d, std::vector<unsigned char>& blob) {
  if (lv.empty() || static_cast<int>(lv.size()) > kTailMaxLevels || nc <= 0) return false;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += (bytes + 15) & ~size_t(15);
    return static_cast<int>(o);
  };
  d = TailDesc{};
  d.nlev = static_cast<int>(lv.size());
  for (int l = 0; l < d.nlev; ++l) {
    const TailLevelHost& h = lv[l];
    TailLevel& L = d.L[l];
    L.m = h.m;
    L.mc = h.mc;
    L.a_ptr = take(4 * h.a_ptr.size());
    L.a_col = take(4 * h.a_col.size());
    L.a_val = take(8 * h.a_val.size());
    L.r_ptr = take(4 * h.r_ptr.size());
    L.r_col = take(4 * h.r_col.size());
    L.r_val = take(8 * h.r_val.size());
    L.p_ptr = take(4 * h.p_ptr.size());
    L.p_col = take(4 * h.p_col.size());
    L.p_val = take(8 * h.p_val.size());
    L.dpre = take(8 * h.dpre.size());
    L.dpost = take(8 * h.dpost.size());
    L.pre_sweeps = h.pre_sweeps;
    L.post_sweeps = h.post_sweeps;
    L.pre_w = h.pre_w;
    L.post_w = h.post_w;
  }
  d.nc = nc;
  d.lu = take(8 * lu.size());
  d.perm = take(4 * perm.size());
  d.blob_bytes = static_cast<int>(off);
  for (int l = 0; l < d.nlev; ++l) {
    TailLevel& L = d.L[l];
    const size_t vb = 8 * static_cast<size_t>(L.m);
    L.vr = take(vb);
    L.vz = take(vb);
    L.vt = take(vb);
    L.v1 = take(vb);
    L.v2 = take(vb);
  }
  d.cr = take(8 * static_cast<size_t>(nc));
  d.cz = take(8 * static_cast<size_t>(nc));
  d.total_bytes = static_cast<int>(off);
  if (off > max_bytes) return false;
  blob.assign(d.blob_bytes, 0);
  auto put = [&](int o, const void* p, size_t bytes) {
    if (bytes) std::memcpy(blob.data() + o, p, bytes);
  };
  for (int l = 0; l < d.nlev; ++l) {
    const TailLevelHost& h = lv[l];
    const TailLevel& L = d.L[l];
    put(L.a_ptr, h.a_ptr.data(), 4 * h.a_ptr.size());
    put(L.a_col, h.a_col.data(), 4 * h.a_col.size());
    put(L.a_val, h.a_val.data(), 8 * h.a_val.size());
    put(L.r_ptr, h.r_ptr.data(), 4 * h.r_ptr.size());
    put(L.r_col, h.r_col.data(), 4 * h.r_col.size());
    put(L.r_val, h.r_val.data(), 8 * h.r_val.size());
    put(L.p_ptr, h.p_ptr.data(), 4 * h.p_ptr.size());
    put(L.p_col, h.p_col.data(), 4 * h.p_col.size());
    put(L.p_val, h.p_val.data(), 8 * h.p_val.size());
    put(L.dpre, h.dpre.data(), 8 * h.dpre.size());
    put(L.dpost, h.dpost.data(), 8 * h.dpost.size());
  }
  put(d.lu, lu.data(), 8 * lu.size());
  put(d.perm, perm.data(), 4 * perm.size());
  return true;
}

void prepare_amg_tail(const TailDesc& d) {
  ensure_smem(reinterpret_cast<const void*>(k_amg_tail), static_cast<size_t>(d.total_bytes));
}

void launch_amg_tail(const TailDesc& d, const unsigned char* blob, const double* r, double* z, cudaStream_t s) {
  launch_pdl(k_amg_tail, 1, kTT, static_cast<size_t>(d.total_bytes), s, d, blob, r, z);
  MGRX_LAUNCH_CK();
  count_launch();
}

}  // namespace mgrx
