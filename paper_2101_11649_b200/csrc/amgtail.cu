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
#include <cstdio>
#include <cstdlib>
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
  // the row sum is a serial chain (left to right); its operands are fetched
  // 4 entries ahead (column, then x and the matrix value), so the chain waits
  // on additions only, not on two dependent shared-memory loads per entry
  for (int i = threadIdx.x; i < m; i += kTT) {
    double s = 0.0;
    const int lo = ptr[i], hi = ptr[i + 1];
    auto ld4 = [&](int k, double (&xv)[4], double (&av)[4]) {
      const int c0 = col[k], c1 = col[k + 1], c2 = col[k + 2], c3 = col[k + 3];
      xv[0] = x[c0], xv[1] = x[c1], xv[2] = x[c2], xv[3] = x[c3];
      av[0] = val[k], av[1] = val[k + 1], av[2] = val[k + 2], av[3] = val[k + 3];
    };
    auto add4 = [&](const double (&xv)[4], const double (&av)[4]) {
      const double q0 = __dmul_rn(av[0], xv[0]), q1 = __dmul_rn(av[1], xv[1]);
      const double q2 = __dmul_rn(av[2], xv[2]), q3 = __dmul_rn(av[3], xv[3]);
      s = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(s, q0), q1), q2), q3);
    };
    double xa[4], aa[4], xb[4], ab[4];
    int k = lo;
    if (k + 4 <= hi) ld4(k, xa, aa);
    while (k + 8 <= hi) {
      ld4(k + 4, xb, ab);
      add4(xa, aa);
      k += 4;
      if (k + 8 <= hi) {
        ld4(k + 4, xa, aa);
        add4(xb, ab);
        k += 4;
      } else {
        add4(xb, ab);
        k += 4;
        goto tail;
      }
    }
    if (k + 4 <= hi) {
      add4(xa, aa);
      k += 4;
    }
  tail:
    for (; k < hi; ++k) s = __dadd_rn(s, __dmul_rn(val[k], x[col[k]]));
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

// ---------------------------------------------------------------------------
// Cluster tail
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned ct_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void ct_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void ct_store_remote(const double* local_addr, unsigned cta, double v) {
  unsigned la = static_cast<unsigned>(__cvta_generic_to_shared(local_addr)), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(cta));
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
}
__host__ __device__ __forceinline__ int ct_lo(int m, int c) {
  return static_cast<int>(static_cast<long long>(m) * c / kCtCtas);
}

struct CtCtx {
  double* full[2];  // replicated gather source, double-buffered
  double* prod;     // products of the current chunk
  int fb;           // buffer holding the most recently published vector
  unsigned rank;
  unsigned phase;            // arrivals so far (ct_arrive_wait)
  volatile unsigned* flags;  // flags[p]: phases CTA p has announced to this CTA
};

// Cluster-wide synchronisation through arrival counters in distributed shared
// memory: after a CTA barrier, 16 threads order the CTA's remote stores
// (fence) and write the new phase number into every peer's flags[rank]; the
// CTA goes on when all 16 of its own counters show that phase. The hardware
// cluster barrier measured ~5 us per use inside this kernel (91 us for its 16
// phases at cfg2, levels 4-6); it is kept for the first and last rendezvous.
__device__ __forceinline__ void ct_arrive_wait(CtCtx& cx) {
  ++cx.phase;
  __syncthreads();
  if (threadIdx.x < kCtCtas) {
    asm volatile("fence.acq_rel.cluster;" ::: "memory");
    unsigned la = static_cast<unsigned>(__cvta_generic_to_shared(const_cast<unsigned*>(cx.flags + cx.rank))), ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(threadIdx.x));
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(ra), "r"(cx.phase) : "memory");
    while (cx.flags[threadIdx.x] < cx.phase) {
    }
    asm volatile("fence.acq_rel.cluster;" ::: "memory");
  }
  __syncthreads();
}

// Push this CTA's slice [lo, hi) of a vector (local[i - lo]) into every CTA's
// spare buffer at index i, then flip buffers behind a cluster barrier.
__device__ __forceinline__ void ct_publish(CtCtx& cx, const double* local, int lo, int hi) {
  double* dst = cx.full[cx.fb ^ 1];
  for (int i = lo + threadIdx.x; i < hi; i += kCtThreads) {
    const double v = local[i - lo];
#pragma unroll
    for (unsigned c = 0; c < kCtCtas; ++c) ct_store_remote(dst + i, c, v);
  }
  ct_arrive_wait(cx);
  cx.fb ^= 1;
}

// One operator as a CTA sees it: its slice of the row pointers (index i - lo)
// and its chunk table in shared memory; entries addressed by their global
// position k (the pointers are rebased when the slice is resident).
struct CtOp {
  const int* ptr;  // shared: ptr[i - lo]
  int lo;
  const int* col;
  const double* val;
  const int* chunks;  // shared: {n, b_0 .. b_n}
};

// epi(i, s) for the rows i of this CTA's slice, s = sum_k val_k x_col_k with x
// the published vector.
template <class Epi>
__device__ __forceinline__ void ct_spmv(const CtCtx& cx, const CtOp& op, Epi epi) {
  const double* x = cx.full[cx.fb];
  const int nch = op.chunks[0];
  const int* __restrict__ col = op.col;
  const double* __restrict__ val = op.val;
  for (int ch = 0; ch < nch; ++ch) {
    const int rs = op.chunks[1 + ch], re = op.chunks[2 + ch];
    const int p0 = op.ptr[rs - op.lo], p1 = op.ptr[re - op.lo];
    const int i = rs + threadIdx.x;
    int lo = 0, hi = 0;
    if (i < re) {
      lo = op.ptr[i - op.lo];
      hi = op.ptr[i + 1 - op.lo];
    }
    // products of the chunk at their entry positions (coalesced operator reads,
    // 8 entries per thread in flight)
    for (int k0 = p0 + threadIdx.x; k0 < p1; k0 += 8 * kCtThreads) {
      int c[8];
      double a[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (k0 + u * kCtThreads < p1) {
          c[u] = col[k0 + u * kCtThreads];
          a[u] = val[k0 + u * kCtThreads];
        }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (k0 + u * kCtThreads < p1) cx.prod[k0 + u * kCtThreads - p0] = __dmul_rn(a[u], x[c[u]]);
    }
    __syncthreads();
    if (i < re) {
      const double* q = cx.prod - p0;
      double s = 0.0;
      int k = lo;
      for (; k + 8 <= hi; k += 8) {
        double t[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) t[u] = q[k + u];
#pragma unroll
        for (int u = 0; u < 8; ++u) s = __dadd_rn(s, t[u]);
      }
      for (; k < hi; ++k) s = __dadd_rn(s, q[k]);
      epi(i, s);
    }
    __syncthreads();
  }
}

// z = S(b) (acc == false) or z += S(b): weighted Jacobi sweeps from zero on
// this CTA's slice [lo, hi); b, z, v: slice-local vectors. The final iterate is
// published (it is the next operation's gather source).
__device__ void ct_jacobi(CtCtx& cx, int lo, int hi, const CtOp& A, const double* dinv /* slice-local */, double w,
                          int sweeps, const double* b, double* z, bool acc, double* v) {
  if (sweeps <= 1) {
    for (int i = lo + threadIdx.x; i < hi; i += kCtThreads) {
      const double t = __dmul_rn(w, __dmul_rn(dinv[i - lo], b[i - lo]));
      z[i - lo] = acc ? __dadd_rn(z[i - lo], t) : t;
    }
    __syncthreads();
    ct_publish(cx, z, lo, hi);
    return;
  }
  for (int i = lo + threadIdx.x; i < hi; i += kCtThreads)
    v[i - lo] = __dmul_rn(w, __dmul_rn(dinv[i - lo], b[i - lo]));
  __syncthreads();
  ct_publish(cx, v, lo, hi);
  for (int sw = 1; sw < sweeps; ++sw) {
    const bool last = sw == sweeps - 1;
    const double* cur = cx.full[cx.fb];
    double* nxt = last ? z : v;
    ct_spmv(cx, A, [&](int i, double s) {
      const double d = __dsub_rn(b[i - lo], __dadd_rn(0.0, s));
      const double t = __dadd_rn(cur[i], __dmul_rn(w, __dmul_rn(dinv[i - lo], d)));
      nxt[i - lo] = (last && acc) ? __dadd_rn(z[i - lo], t) : t;
    });
    ct_publish(cx, nxt, lo, hi);
  }
}

__global__ void __launch_bounds__(kCtThreads, 1)
    k_amg_ctail(TailDesc d, CtLayout lay, const unsigned char* __restrict__ blob, const double* __restrict__ r,
                double* __restrict__ z) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int T = threadIdx.x;
  __shared__ unsigned ct_flags[kCtCtas];
  if (T < kCtCtas) ct_flags[T] = 0u;
  CtCtx cx;
  cx.rank = ct_rank();
  cx.fb = 0;
  cx.phase = 0;
  cx.flags = ct_flags;
  cx.full[0] = reinterpret_cast<double*>(sm + lay.full0);
  cx.full[1] = reinterpret_cast<double*>(sm + lay.full1);
  cx.prod = reinterpret_cast<double*>(sm + lay.prod);
  const unsigned c = cx.rank;
  auto B = [&](int o) { return blob + o; };
  // ---- prologue (setup data only, before the previous kernel is waited for):
  // chunk tables and row-pointer slices, then the resident entry slices
  CtOp opA[kTailMaxLevels], opR[kTailMaxLevels], opP[kTailMaxLevels];
  auto stage_meta = [&](CtOp& op, const CtMat& ml, int gptr, int gchunks, int rows) {
    const int lo = ct_lo(rows, c), hi = ct_lo(rows, c + 1);
    int* sp = reinterpret_cast<int*>(sm + ml.ptr);
    int* sc = reinterpret_cast<int*>(sm + ml.chunks);
    const int* gp = reinterpret_cast<const int*>(B(gptr));
    const int* gc = reinterpret_cast<const int*>(B(gchunks)) + static_cast<size_t>(c) * (kCtMaxChunks + 2);
    for (int i = T; i <= hi - lo; i += kCtThreads) sp[i] = gp[lo + i];
    for (int i = T; i < kCtMaxChunks + 2; i += kCtThreads) sc[i] = gc[i];
    op.ptr = sp;
    op.lo = lo;
    op.chunks = sc;
  };
  for (int l = 0; l < d.nlev; ++l) {
    stage_meta(opA[l], lay.A[l], d.L[l].a_ptr, d.L[l].a_chunks, d.L[l].m);
    stage_meta(opR[l], lay.R[l], d.L[l].r_ptr, d.L[l].r_chunks, d.L[l].mc);
    stage_meta(opP[l], lay.P[l], d.L[l].p_ptr, d.L[l].p_chunks, d.L[l].m);
  }
  __syncthreads();
  auto stage_entries = [&](CtOp& op, const CtMat& ml, int gcol, int gval, int rows) {
    const int lo = ct_lo(rows, c), hi = ct_lo(rows, c + 1);
    const int p0 = op.ptr[0], p1 = op.ptr[hi - lo];
    const int* gc = reinterpret_cast<const int*>(B(gcol));
    const double* gv = reinterpret_cast<const double*>(B(gval));
    if (ml.col >= 0) {
      int* scol = reinterpret_cast<int*>(sm + ml.col);
      double* sval = reinterpret_cast<double*>(sm + ml.val);
      for (int k = p0 + T; k < p1; k += kCtThreads) {
        scol[k - p0] = gc[k];
        sval[k - p0] = gv[k];
      }
      op.col = scol - p0;
      op.val = sval - p0;
    } else {
      op.col = gc;
      op.val = gv;
    }
  };
  for (int l = 0; l < d.nlev; ++l) {
    const int lo = ct_lo(d.L[l].m, c), hi = ct_lo(d.L[l].m, c + 1);
    const double* gpre = reinterpret_cast<const double*>(B(d.L[l].dpre));
    const double* gpost = reinterpret_cast<const double*>(B(d.L[l].dpost));
    double* spre = reinterpret_cast<double*>(sm + lay.dpre[l]);
    double* spost = reinterpret_cast<double*>(sm + lay.dpost[l]);
    for (int i = lo + T; i < hi; i += kCtThreads) {
      spre[i - lo] = gpre[i];
      spost[i - lo] = gpost[i];
    }
    stage_entries(opA[l], lay.A[l], d.L[l].a_col, d.L[l].a_val, d.L[l].m);
    stage_entries(opR[l], lay.R[l], d.L[l].r_col, d.L[l].r_val, d.L[l].mc);
    stage_entries(opP[l], lay.P[l], d.L[l].p_col, d.L[l].p_val, d.L[l].m);
  }
  double* vr[kTailMaxLevels + 1];
  double *vz[kTailMaxLevels], *vt[kTailMaxLevels], *vv[kTailMaxLevels];
  for (int l = 0; l < d.nlev; ++l) {
    vr[l] = reinterpret_cast<double*>(sm + lay.vr[l]);
    vz[l] = reinterpret_cast<double*>(sm + lay.vz[l]);
    vt[l] = reinterpret_cast<double*>(sm + lay.vt[l]);
    vv[l] = reinterpret_cast<double*>(sm + lay.vv[l]);
  }
  vr[d.nlev] = reinterpret_cast<double*>(sm + lay.vr[d.nlev]);
  pdl_enter();  // r is the previous kernel's
  {
    const int lo = ct_lo(d.L[0].m, c), hi = ct_lo(d.L[0].m, c + 1);
    for (int i = lo + T; i < hi; i += kCtThreads) vr[0][i - lo] = r[i];
  }
  __syncthreads();
  ct_sync();  // every CTA of the cluster is running before any remote store
  // down
  for (int l = 0; l < d.nlev; ++l) {
    const TailLevel& L = d.L[l];
    const int lo = ct_lo(L.m, c), hi = ct_lo(L.m, c + 1);
    double *rl = vr[l], *zl = vz[l], *tl = vt[l];
    ct_jacobi(cx, lo, hi, opA[l], reinterpret_cast<const double*>(sm + lay.dpre[l]), L.pre_w, L.pre_sweeps, rl, zl,
              false, vv[l]);
    ct_spmv(cx, opA[l], [&](int i, double s) { tl[i - lo] = __dsub_rn(rl[i - lo], __dadd_rn(0.0, s)); });
    ct_publish(cx, tl, lo, hi);
    const int nlo = ct_lo(L.mc, c);
    double* rn = vr[l + 1];
    ct_spmv(cx, opR[l], [&](int i, double s) { rn[i - nlo] = __dadd_rn(0.0, s); });
  }
  // coarsest: the right-hand side is published, CTA 0's first warp solves in
  // the dense algorithm's order (DenseLU) and pushes the solution to all
  {
    const int n = d.nc;
    ct_publish(cx, vr[d.nlev], ct_lo(n, c), ct_lo(n, c + 1));
    if (c == 0 && T < 32) {
      // factors into shared memory first (one coalesced pass): the 2n steps
      // below are then short dependent shared-memory steps
      const double* Mg = reinterpret_cast<const double*>(B(d.lu));
      const int* pm = reinterpret_cast<const int*>(B(d.perm));
      const double* rc = cx.full[cx.fb];
      double* M = cx.prod;
      double* xs = cx.prod + static_cast<size_t>(n) * n;
      for (int i = T; i < n * n; i += 32) M[i] = Mg[i];
      for (int i = T; i < n; i += 32) xs[i] = rc[pm[i]];
      __syncwarp();
      for (int j = 0; j < n; ++j) {
        const double xj = xs[j];
        for (int i = j + 1 + T; i < n; i += 32)
          xs[i] = __dsub_rn(xs[i], __dmul_rn(M[static_cast<size_t>(j) * n + i], xj));
        __syncwarp();
      }
      for (int j = n - 1; j >= 0; --j) {
        if (T == 0) xs[j] = __ddiv_rn(xs[j], M[static_cast<size_t>(j) * n + j]);
        __syncwarp();
        const double xj = xs[j];
        for (int i = T; i < j; i += 32) xs[i] = __dsub_rn(xs[i], __dmul_rn(M[static_cast<size_t>(j) * n + i], xj));
        __syncwarp();
      }
      double* dst = cx.full[cx.fb ^ 1];
      for (int i = T; i < n; i += 32) {
        const double v = xs[i];
#pragma unroll
        for (unsigned cc = 0; cc < kCtCtas; ++cc) ct_store_remote(dst + i, cc, v);
      }
    }
    ct_arrive_wait(cx);
    cx.fb ^= 1;
  }
  // up
  for (int l = d.nlev - 1; l >= 0; --l) {
    const TailLevel& L = d.L[l];
    const int lo = ct_lo(L.m, c), hi = ct_lo(L.m, c + 1);
    double *rl = vr[l], *zl = vz[l], *tl = vt[l];
    // z += P e (e = the deeper level's published solution)
    ct_spmv(cx, opP[l], [&](int i, double s) { zl[i - lo] = __dadd_rn(zl[i - lo], s); });
    ct_publish(cx, zl, lo, hi);
    ct_spmv(cx, opA[l], [&](int i, double s) { tl[i - lo] = __dsub_rn(rl[i - lo], __dadd_rn(0.0, s)); });
    ct_jacobi(cx, lo, hi, opA[l], reinterpret_cast<const double*>(sm + lay.dpost[l]), L.post_w, L.post_sweeps, tl,
              zl, true, vv[l]);
  }
  {
    const int lo = ct_lo(d.L[0].m, c), hi = ct_lo(d.L[0].m, c + 1);
    for (int i = lo + T; i < hi; i += kCtThreads) z[i] = vz[0][i - lo];
  }
  ct_sync();  // no CTA exits while a peer may still address its shared memory
}

}  // namespace

bool build_ctail_blob(const std::vector<TailLevelHost>& lv, int nc, const std::vector<double>& lu,
                      const std::vector<int>& perm, TailDesc& d, std::vector<unsigned char>& blob, CtLayout& lay) {
  if (lv.empty() || lv[0].m > kCtMaxRows || static_cast<long long>(nc) * nc + nc > kCtProd) return false;
  if (!build_tail_blob(lv, nc, lu, perm, size_t(1) << 30, d, blob)) return false;
  // per-CTA row chunk tables: {n, b_0 .. b_n} with <= kCtProd entries per chunk
  bool ok = true;
  auto table = [&](const std::vector<int>& ptr, int rows) {
    std::vector<int> t(static_cast<size_t>(kCtCtas) * (kCtMaxChunks + 2), 0);
    for (int c = 0; c < kCtCtas; ++c) {
      int* e = t.data() + static_cast<size_t>(c) * (kCtMaxChunks + 2);
      const int lo = ct_lo(rows, c), hi = ct_lo(rows, c + 1);
      int n = 0, rs = lo;
      e[1] = lo;
      while (rs < hi) {
        int re = rs;
        // (a chunk also holds at most one row per thread)
        while (re < hi && re - rs < kCtThreads && ptr[re + 1] - ptr[rs] <= kCtProd) ++re;
        if (re == rs || n == kCtMaxChunks) {
          ok = false;
          return t;
        }
        e[2 + n] = re;
        ++n;
        rs = re;
      }
      e[0] = n;
    }
    return t;
  };
  auto append = [&](const std::vector<int>& t) {
    const size_t o = (blob.size() + 15) & ~size_t(15);
    blob.resize(o + 4 * t.size());
    std::memcpy(blob.data() + o, t.data(), 4 * t.size());
    return static_cast<int>(o);
  };
  for (size_t l = 0; l < lv.size(); ++l) {
    d.L[l].a_chunks = append(table(lv[l].a_ptr, lv[l].m));
    d.L[l].r_chunks = append(table(lv[l].r_ptr, lv[l].mc));
    d.L[l].p_chunks = append(table(lv[l].p_ptr, lv[l].m));
  }
  if (!ok) return false;
  // shared-memory layout
  lay = CtLayout{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += (bytes + 15) & ~size_t(15);
    return static_cast<int>(o);
  };
  lay.full0 = take(8 * static_cast<size_t>(lv[0].m));
  lay.full1 = take(8 * static_cast<size_t>(lv[0].m));
  lay.prod = take(8 * static_cast<size_t>(kCtProd));
  auto slice = [](int rows) { return static_cast<size_t>(rows / kCtCtas + 2); };
  for (size_t l = 0; l < lv.size(); ++l) {
    if (lv[l].m > lv[0].m || lv[l].mc > lv[0].m) return false;
    lay.vr[l] = take(8 * slice(lv[l].m));
    lay.vz[l] = take(8 * slice(lv[l].m));
    lay.vt[l] = take(8 * slice(lv[l].m));
    lay.vv[l] = take(8 * slice(lv[l].m));
    lay.dpre[l] = take(8 * slice(lv[l].m));
    lay.dpost[l] = take(8 * slice(lv[l].m));
  }
  lay.vr[lv.size()] = take(8 * slice(nc));
  for (size_t l = 0; l < lv.size(); ++l) {
    lay.A[l].ptr = take(4 * (slice(lv[l].m) + 1));
    lay.A[l].chunks = take(4 * (kCtMaxChunks + 2));
    lay.R[l].ptr = take(4 * (slice(lv[l].mc) + 1));
    lay.R[l].chunks = take(4 * (kCtMaxChunks + 2));
    lay.P[l].ptr = take(4 * (slice(lv[l].m) + 1));
    lay.P[l].chunks = take(4 * (kCtMaxChunks + 2));
  }
  constexpr size_t kBudget = 224 * 1024;
  if (off > kBudget) return false;
  // resident entry slices, deepest levels first (they are the latency-bound ones)
  auto max_slice_entries = [&](const std::vector<int>& ptr, int rows) {
    int mx = 0;
    for (int c = 0; c < kCtCtas; ++c) mx = std::max(mx, ptr[ct_lo(rows, c + 1)] - ptr[ct_lo(rows, c)]);
    return static_cast<size_t>(mx);
  };
  auto try_res = [&](CtMat& ml, const std::vector<int>& ptr, int rows) {
    const size_t e = max_slice_entries(ptr, rows);
    const size_t need = ((4 * e + 15) & ~size_t(15)) + ((8 * e + 15) & ~size_t(15));
    if (off + need > kBudget) return;
    ml.col = take(4 * e);
    ml.val = take(8 * e);
  };
  for (int l = static_cast<int>(lv.size()) - 1; l >= 0; --l) {
    try_res(lay.A[l], lv[l].a_ptr, lv[l].m);
    try_res(lay.R[l], lv[l].r_ptr, lv[l].mc);
    try_res(lay.P[l], lv[l].p_ptr, lv[l].m);
  }
  lay.total = static_cast<int>(off);
  return true;
}

void prepare_amg_ctail(const CtLayout& lay) {
  const void* k = reinterpret_cast<const void*>(k_amg_ctail);
  ensure_smem(k, static_cast<size_t>(lay.total));
  if (first_on_device(reinterpret_cast<const char*>(k) + 1))
    MGRX_CK(cudaFuncSetAttribute(k_amg_ctail, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
}

void launch_amg_ctail(const TailDesc& d, const CtLayout& lay, const unsigned char* blob, const double* r, double* z,
                      cudaStream_t s) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(kCtCtas);
  cfg.blockDim = dim3(kCtThreads);
  cfg.dynamicSmemBytes = static_cast<size_t>(lay.total);
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() && !kPdlStagedEarly ? 1 : 0;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = kCtCtas;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  MGRX_CK(cudaLaunchKernelEx(&cfg, k_amg_ctail, d, lay, blob, r, z));
  count_launch();
}

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
