// Device hierarchies. Setup follows proj/src/mgr.cpp:223-316 and
// proj/src/amg.cpp:147-291 step by step, with every matrix built by the
// bit-exact kernels of sparse.cu / coarsen.cu. Application follows
// proj/src/mgr.cpp:177-219 and proj/src/amg.cpp:232-242 with the fusions
// documented inline (each one preserves the reference's arithmetic).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <unordered_set>

#include "coarsen.cuh"
#include "hierarchy.cuh"
#include "krylov.cuh"

#include <cstring>
#include <functional>

namespace mgrx {
namespace {

__global__ void k_split(int n, const int* __restrict__ labels, const uint8_t* __restrict__ mask,
                        uint8_t* __restrict__ isf, uint8_t* __restrict__ isc) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint8_t f = mask[labels[i]];
  isf[i] = f;
  isc[i] = f ? 0 : 1;
}

__global__ void k_gather_int(int n, const int* __restrict__ idx, const int* __restrict__ in,
                             int* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[idx[i]];
}

__global__ void k_scatter_add(int n, const int* __restrict__ idx, const double* __restrict__ a,
                              double* __restrict__ z) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) z[idx[i]] = __dadd_rn(z[idx[i]], a[i]);
}

// P = [-W; I] in global order with W = A_FC scaled by dinv_F
// (proj/src/mgr.cpp:89-114): C rows carry (cpos, 1.0); F rows carry
// -(a_fc * dinv_f) at the coarse positions of their C columns.
template <bool kFill>
__global__ void k_mgr_interp(int n, const int* __restrict__ ptr, const int* __restrict__ col,
                             const double* __restrict__ val, const int* __restrict__ fpos,
                             const int* __restrict__ cpos, const double* __restrict__ dinv_f,
                             int* __restrict__ cnt, const int* __restrict__ optr,
                             int* __restrict__ ocol, double* __restrict__ oval) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  if (cpos[r] >= 0) {
    if (kFill) {
      ocol[optr[r]] = cpos[r];
      oval[optr[r]] = 1.0;
    } else {
      cnt[r] = 1;
    }
    return;
  }
  const double dv = kFill ? dinv_f[fpos[r]] : 0.0;
  int o = kFill ? optr[r] : 0;
  int c = 0;
  for (int k = ptr[r]; k < ptr[r + 1]; ++k) {
    const int j = cpos[col[k]];
    if (j < 0) continue;
    if (kFill) {
      ocol[o] = j;
      oval[o] = -__dmul_rn(val[k], dv);
      ++o;
    }
    ++c;
  }
  if (!kFill) cnt[r] = c;
}

// R rows span C (proj/src/mgr.cpp:116-146). Injection: (C[j], 1). Jacobi /
// ideal-with-diagonal-A_FF: -(a_cf * dinv_f) at global F columns plus
// (C[j], 1), merged in column order.
template <bool kFill>
__global__ void k_mgr_restrict(int nc, bool injection, const int* __restrict__ ptr,
                               const int* __restrict__ col, const double* __restrict__ val,
                               const int* __restrict__ C, const int* __restrict__ fpos,
                               const double* __restrict__ dinv_f, int* __restrict__ cnt,
                               const int* __restrict__ optr, int* __restrict__ ocol,
                               double* __restrict__ oval) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nc) return;
  const int r = C[j];
  int o = kFill ? optr[j] : 0;
  int c = 0;
  bool placed = false;
  auto emit = [&](int cc, double v) {
    if (kFill) {
      ocol[o] = cc;
      oval[o] = v;
      ++o;
    }
    ++c;
  };
  if (!injection) {
    for (int k = ptr[r]; k < ptr[r + 1]; ++k) {
      const int g = col[k];
      if (!placed && g > r) {
        emit(r, 1.0);
        placed = true;
      }
      const int f = fpos[g];
      if (f >= 0) emit(g, kFill ? -__dmul_rn(val[k], dinv_f[f]) : 0.0);
    }
  }
  if (!placed) emit(r, 1.0);
  if (!kFill) cnt[j] = c;
}

// P from W = A_FF^{-1} A_FC (ideal interpolation through a block or dense
// solve): F rows -W(fpos, :), C rows the identity (build_interp,
// proj/src/mgr.cpp:105-113).
template <bool kFill>
__global__ void k_interp_from_w(int n, const int* __restrict__ fpos, const int* __restrict__ cpos,
                                const int* __restrict__ wptr, const int* __restrict__ wcol,
                                const double* __restrict__ wval, int* __restrict__ cnt,
                                const int* __restrict__ optr, int* __restrict__ ocol, double* __restrict__ oval) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  if (cpos[r] >= 0) {
    if (kFill) {
      ocol[optr[r]] = cpos[r];
      oval[optr[r]] = 1.0;
    } else {
      cnt[r] = 1;
    }
    return;
  }
  const int f = fpos[r];
  if (!kFill) {
    cnt[r] = wptr[f + 1] - wptr[f];
    return;
  }
  int o = optr[r];
  for (int k = wptr[f]; k < wptr[f + 1]; ++k, ++o) {
    ocol[o] = wcol[k];
    oval[o] = -wval[k];
  }
}

// R from Z = A_CF A_FF^{-1} (ideal restriction): row j holds -Z(j, :) at the
// global F columns and (C[j], 1), in column order (proj/src/mgr.cpp:137-145).
template <bool kFill>
__global__ void k_restrict_from_z(int nc, const int* __restrict__ C, const int* __restrict__ F,
                                  const int* __restrict__ zptr, const int* __restrict__ zcol,
                                  const double* __restrict__ zval, int* __restrict__ cnt,
                                  const int* __restrict__ optr, int* __restrict__ ocol, double* __restrict__ oval) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nc) return;
  if (!kFill) {
    cnt[j] = zptr[j + 1] - zptr[j] + 1;
    return;
  }
  const int r = C[j];
  int o = optr[j];
  bool placed = false;
  for (int k = zptr[j]; k < zptr[j + 1]; ++k) {
    const int g = F[zcol[k]];
    if (!placed && g > r) {
      ocol[o] = r;
      oval[o++] = 1.0;
      placed = true;
    }
    ocol[o] = g;
    oval[o++] = -zval[k];
  }
  if (!placed) {
    ocol[o] = r;
    oval[o] = 1.0;
  }
}

// X = A_FF^{-1} B by the exact routes of ff_inverse_times
// (proj/src/mgr.cpp:46-65) other than the structurally diagonal one.
DCsr ff_solve(const DCsr& Aff, const DCsr& B, const std::optional<std::vector<int>>& layout, cudaStream_t s) {
  if (layout) {
    BlockLU f;
    block_factor(Aff, *layout, f, s);
    return block_solve_columns(f, B, s);
  }
  if (Aff.rows <= 2000) {
    DenseLU f;
    dense_factor(Aff, f, s, 1e-300, false);
    return dense_solve_columns(f, B, s);
  }
  throw RuntimeError(
      "ideal transfer operators require a structurally diagonal A_FF, a declared block "
      "layout, or |F| <= 2000 for a dense factorization");
}

__global__ void k_scatter_count(int m, const int* __restrict__ idx, const int* __restrict__ sptr,
                                int* __restrict__ cnt) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < m) cnt[idx[r]] = sptr[r + 1] - sptr[r];
}

// Unknown-based P assembly (proj/src/amg.cpp:201-222): sub-row r of a group
// becomes global row idx[r]; local coarse column k maps to the rank of its
// global fine index among all C points.
__global__ void k_group_fill(int m, const int* __restrict__ idx, const int* __restrict__ csub,
                             const int* __restrict__ cid_global, const int* __restrict__ sptr,
                             const int* __restrict__ scol, const double* __restrict__ sval,
                             const int* __restrict__ optr, int* __restrict__ ocol,
                             double* __restrict__ oval) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  int o = optr[idx[r]];
  for (int k = sptr[r]; k < sptr[r + 1]; ++k, ++o) {
    ocol[o] = cid_global[idx[csub[scol[k]]]];
    oval[o] = sval[k];
  }
}

__global__ void k_mark_group_c(int m, const int* __restrict__ idx, const uint8_t* __restrict__ sub_c,
                               uint8_t* __restrict__ is_c) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < m && sub_c[r]) is_c[idx[r]] = 1;
}

__global__ void k_eq_flag(int n, const int* __restrict__ a, int v, uint8_t* __restrict__ f) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) f[i] = a[i] == v ? 1 : 0;
}
__global__ void k_not(int n, const uint8_t* __restrict__ a, uint8_t* __restrict__ f) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) f[i] = a[i] ? 0 : 1;
}

template <class K, class... Args>
void launch1d(K kern, int n, cudaStream_t s, Args... args) {
  if (n <= 0) return;
  kern<<<blocks_for(n, 256), 256, 0, s>>>(n, args...);
  MGRX_LAUNCH_CK();
  count_launch();
}

std::vector<int> gather_host(const std::vector<int>& v, const std::vector<int>& idx) {
  std::vector<int> o;
  o.reserve(idx.size());
  for (int i : idx) o.push_back(v[i]);
  return o;
}

}  // namespace

// ============================================================================
// BoundRelax
// ============================================================================
void BoundRelax::bind(const SmootherSpec& s, const DCsr& mat, const std::vector<int>* umap,
                      cudaStream_t st) {
  if (mat.rows != mat.cols) throw InvalidArgument("smoother: matrix must be square");
  if (s.sweeps < 1) throw InvalidArgument("smoother: sweeps must be >= 1");
  if (!(s.weight > 0.0 && s.weight < 2.0)) throw InvalidArgument("smoother: weight must lie in (0, 2)");
  spec = s;
  A = &mat;
  n = mat.rows;
  switch (s.kind) {
    case Smoother::jacobi:
      diag_inverse(mat, dinv, st);
      break;
    case Smoother::l1_jacobi: {
      DVec<double> d;
      l1_diagonal(mat, true, d, st);
      dinv.alloc(n > 0 ? n : 1, st);
      reciprocal(n, d.get(), dinv.get(), st);  // proj/src/relax.cpp:106-113
      break;
    }
    case Smoother::hybrid_l1_gs_forward:
    case Smoother::hybrid_l1_gs_backward: {
      // Normalise the partition exactly like proj/src/relax.cpp:12-23. With
      // several ranges, rows read the snapshot across ranges: the sweep's
      // dependencies and the L1 diagonal follow the range owner of each row.
      const int* own = nullptr;
      if (!s.partition.empty()) {
        int expect = 0;
        for (const auto& [b, e] : s.partition) {
          if (b != expect || e <= b)
            throw InvalidArgument("smoother partition ranges must tile [0,n) in order");
          expect = e;
        }
        if (expect != n) throw InvalidArgument("smoother partition does not cover the matrix");
        if (s.partition.size() > 1) {
          std::vector<int> ho(n);
          for (int k = 0; k < static_cast<int>(s.partition.size()); ++k)
            for (int i = s.partition[k].first; i < s.partition[k].second; ++i) ho[i] = k;
          owner.alloc(n, st);
          owner.upload(ho.data(), n);
          own = owner.get();
        }
      }
      l1_diagonal(mat, false, l1d, st, own);
      gs_schedule(mat, s.kind == Smoother::hybrid_l1_gs_forward, l1d.get(), s.sweeps > 1, sched, st, own);
      gs_bind_scratch(gs, st);
      break;
    }
    case Smoother::block_jacobi_exact:
      // proj/src/relax.cpp:126-131, block LU per diagonal block
      if (s.block_sizes.empty()) throw InvalidArgument("smoother: block_jacobi_exact requires block sizes");
      block_factor(mat, s.block_sizes, blk, st);
      break;
    case Smoother::dense_lu:
      dense_factor(mat, lu, st);
      break;
    case Smoother::amg_vcycle: {
      AmgSpec cfg = s.amg ? *s.amg : AmgSpec{};
      std::vector<int> um;
      if (s.use_unknown_map) {
        if (umap == nullptr)
          throw InvalidArgument("smoother: use_unknown_map set but no unknown map supplied");
        um = *umap;
      }
      amg = std::make_unique<AmgHier>();
      amg->setup(mat, cfg, um, st);
      break;
    }
  }
  w0.alloc(n > 0 ? n : 1, st);
  if (s.sweeps > 1 || s.kind == Smoother::amg_vcycle) {
    w1.alloc(n > 0 ? n : 1, st);
    w2.alloc(n > 0 ? n : 1, st);
  }
}

void BoundRelax::apply(const double* r, const int* rrow, double* z, cudaStream_t st) {
  if (n == 0) return;
  const double* rc = r;
  if (rrow && (spec.kind != Smoother::jacobi && spec.kind != Smoother::l1_jacobi)) {
    gather(n, rrow, r, w0.get(), st);
    rc = w0.get();
    rrow = nullptr;
  }
  switch (spec.kind) {
    case Smoother::dense_lu:
      dense_solve(lu, rc, z, st);
      return;
    case Smoother::block_jacobi_exact:
      block_solve(blk, rc, z, st);
      return;
    case Smoother::jacobi:
    case Smoother::l1_jacobi:
      jacobi_sweeps(rc, rrow, z, nullptr, st);
      return;
    case Smoother::hybrid_l1_gs_forward:
    case Smoother::hybrid_l1_gs_backward: {
      const bool fwd = spec.kind == Smoother::hybrid_l1_gs_forward;
      const double* xold = nullptr;
      double* bufs[2] = {w1.get(), w2.get()};
      for (int sw = 0; sw < spec.sweeps; ++sw) {
        double* xnew = (sw == spec.sweeps - 1) ? z : bufs[sw % 2];
        gs_sweep(*A, sched, l1d.get(), rc, xold, xnew, nullptr, fwd, gs, st);
        xold = xnew;
      }
      return;
    }
    case Smoother::amg_vcycle: {
      // z = V(r); z += V(r - A z) for later sweeps (relax.cpp:186-190)
      amg->vcycle(rc, z, st);
      for (int sw = 1; sw < spec.sweeps; ++sw) {
        spmv_residual(*A, z, rc, nullptr, w1.get(), st);
        amg->vcycle(w1.get(), w2.get(), st);
        vec_add(n, w2.get(), z, st);
      }
      return;
    }
    default:
      throw RuntimeError("smoother: kind not supported on the device path");
  }
}

int fold_sweep0_max_rows() {
  static const int m = [] {
    const char* v = std::getenv("MGRX_FOLD_MAX");
    return v ? std::atoi(v) : 65536;
  }();
  return m;
}

// sweep 0: z = w*(dinv*r); later: z += w*(dinv*(r - A z)) (relax.cpp:168-174).
// Sweep 0 is folded into sweep 1 (its iterate is formed on the fly from r),
// and with zacc the last sweep adds its result into zacc (apply_add).
bool BoundRelax::z0_fusable() const {
  static const bool on = [] {
    const char* v = std::getenv("MGRX_FUSE_J0");
    return !v || std::atoi(v) != 0;
  }();
  // (short rows only: on the long-row levels of cfg4 the extra epilogue
  // traffic of the sum-bound staged kernel measured slower)
  return on && (spec.kind == Smoother::jacobi || spec.kind == Smoother::l1_jacobi) && spec.sweeps >= 2 &&
         (n > fold_sweep0_max_rows() || (A && A->xt_nblk > 0)) && A &&
         static_cast<long long>(A->nnz) <= 24LL * A->rows;
}

void BoundRelax::jacobi_sweeps(const double* rc, const int* rrow, double* z, double* zacc, cudaStream_t st,
                               bool have_z0) {
  if (spec.sweeps <= 1) {
    double* out = zacc ? w0.get() : z;
    jacobi0(n, spec.weight, dinv.get(), rc, rrow, out, st);
    if (zacc) vec_add(n, out, zacc, st);
    return;
  }
  // Folding sweep 0 doubles the gathers per nonzero (dinv and r instead of
  // z): a win only where launch latency dominates (measured at cfg2: levels of
  // <= 64K rows faster, the 1M / 366K-row levels 15-20% slower).
  const double* cur = nullptr;
  double* bufs[2] = {w1.get(), w2.get()};
  // (levels served by the x-window SpMV keep sweep 0 apart too: that kernel
  // stages plain x vectors, not an iterate formed on the fly)
  if (n > fold_sweep0_max_rows() || A->xt_nblk > 0) {
    if (!have_z0) jacobi0(n, spec.weight, dinv.get(), rc, rrow, w2.get(), st);
    cur = w2.get();
    bufs[1] = w0.get();  // w2 holds sweep 0; w0 is free (no gather when jacobi)
  }
  for (int sw = 1; sw < spec.sweeps; ++sw) {
    const bool last = sw == spec.sweeps - 1;
    double* nxt = last ? (zacc ? nullptr : z) : bufs[sw % 2];
    spmv_jacobi_ex(*A, cur, rc, rrow, dinv.get(), spec.weight, nxt, last ? zacc : nullptr, st);
    cur = nxt;
  }
}

void BoundRelax::apply_add(const double* r, double* zacc, cudaStream_t st) {
  if (n == 0) return;
  if (spec.kind == Smoother::jacobi || spec.kind == Smoother::l1_jacobi) {
    jacobi_sweeps(r, nullptr, nullptr, zacc, st);
    return;
  }
  if ((spec.kind == Smoother::hybrid_l1_gs_forward || spec.kind == Smoother::hybrid_l1_gs_backward) &&
      spec.sweeps == 1) {
    gs_sweep(*A, sched, l1d.get(), r, nullptr, w0.get(), zacc,
             spec.kind == Smoother::hybrid_l1_gs_forward, gs, st);
    return;
  }
  apply(r, nullptr, w0.get(), st);
  vec_add(n, w0.get(), zacc, st);
}

void BoundRelax::check(cudaStream_t st) {
  gs_check(gs, st);
  if (amg)
    for (auto& L : amg->levels) {
      L.pre.check(st);
      L.post.check(st);
    }
}

// ============================================================================
// AMG (proj/src/amg.cpp:147-297)
// ============================================================================
namespace {

struct LevelBuild {
  DCsr P;
  DVec<int> C, F;
  std::vector<int> coarse_umap;
  bool stalled = false;
};

LevelBuild build_level_interp(const DCsr& A, double theta, const std::vector<int>& umap,
                              long long* fallback, cudaStream_t s) {
  const int n = A.rows;
  LevelBuild out;
  if (umap.empty()) {
    const DCsr S = strength_graph(A, theta, s);
    DVec<uint8_t> is_c;
    pmis(S, is_c, s);
    DVec<int> cid;
    const int nc = rank_flags(is_c.get(), n, cid, s);
    if (nc == n) {
      out.stalled = true;
      return out;
    }
    out.P = classical_interp(A, S, cid.get(), nc, fallback, s);
    select_flagged(is_c.get(), n, out.C, s);
    DVec<uint8_t> isf(n, s);
    launch1d(k_not, n, s, is_c.get(), isf.get());
    select_flagged(isf.get(), n, out.F, s);
    return out;
  }
  // Unknown-based: per unknown id (ascending), coarsen the extracted
  // sub-block; interpolation never crosses unknowns (amg.cpp:188-200).
  std::vector<int> ids = umap;
  std::sort(ids.begin(), ids.end());
  ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
  DVec<int> dmap(n, s);
  dmap.upload(umap.data(), n);
  DVec<uint8_t> is_c(n, s), flag(n, s);
  is_c.zero();
  struct Group {
    DVec<int> idx, csub;
    DCsr P;
  };
  std::vector<Group> groups(ids.size());
  for (size_t g = 0; g < ids.size(); ++g) {
    launch1d(k_eq_flag, n, s, dmap.get(), ids[g], flag.get());
    const int m = select_flagged(flag.get(), n, groups[g].idx, s);
    const DCsr Asub = extract(A, groups[g].idx.get(), m, groups[g].idx.get(), m, s);
    const DCsr S = strength_graph(Asub, theta, s);
    DVec<uint8_t> sub_c;
    pmis(S, sub_c, s);
    DVec<int> cid;
    const int nc = rank_flags(sub_c.get(), m, cid, s);
    groups[g].P = classical_interp(Asub, S, cid.get(), nc, fallback, s);
    select_flagged(sub_c.get(), m, groups[g].csub, s);
    launch1d(k_mark_group_c, m, s, groups[g].idx.get(), sub_c.get(), is_c.get());
  }
  DVec<int> cid_global;
  const int nc = rank_flags(is_c.get(), n, cid_global, s);
  if (nc == n) {
    out.stalled = true;
    return out;
  }
  DVec<int> cnt(n, s);
  cnt.zero();
  for (auto& g : groups)
    launch1d(k_scatter_count, g.P.rows, s, g.idx.get(), g.P.ptr.get(), cnt.get());
  out.P.rows = n;
  out.P.cols = nc;
  out.P.ptr.alloc(n + 1, s);
  out.P.nnz = static_cast<int>(exclusive_scan(cnt.get(), out.P.ptr.get(), n, s));
  out.P.col.alloc(out.P.nnz, s);
  out.P.val.alloc(out.P.nnz, s);
  for (auto& g : groups)
    launch1d(k_group_fill, g.P.rows, s, g.idx.get(), g.csub.get(), cid_global.get(), g.P.ptr.get(),
             g.P.col.get(), g.P.val.get(), out.P.ptr.get(), out.P.col.get(), out.P.val.get());
  select_flagged(is_c.get(), n, out.C, s);
  DVec<uint8_t> isf(n, s);
  launch1d(k_not, n, s, is_c.get(), isf.get());
  select_flagged(isf.get(), n, out.F, s);
  const std::vector<int> ch = out.C.download(nc);
  out.coarse_umap = gather_host(umap, ch);
  return out;
}

}  // namespace

void AmgHier::setup(const DCsr& A, const AmgSpec& cfg, const std::vector<int>& umap, cudaStream_t s) {
  NvtxRange nvtx("mgrx.amg_setup");
  if (A.rows != A.cols) throw InvalidArgument("amg_setup: matrix must be square");
  if (!(cfg.strength_theta > 0.0 && cfg.strength_theta < 1.0))
    throw InvalidArgument("amg_setup: strength_theta must lie in (0,1)");
  if (cfg.coarse_size < 1) throw InvalidArgument("amg_setup: coarse_size must be >= 1");
  if (!umap.empty() && static_cast<int>(umap.size()) != A.rows)
    throw InvalidArgument("amg_setup: unknown_map size mismatch");
  spec = cfg;
  levels.clear();
  level_sizes.clear();
  DCsr Acur = csr_copy(A, s);
  std::vector<int> map = umap;
  while (true) {
    const int n = Acur.rows;
    level_sizes.push_back(n);
    levels.emplace_back();
    NvtxRange nvtx_level("mgrx.amg_setup.level", static_cast<int>(levels.size()) - 1);
    AmgLevelD& L = levels.back();
    L.umap = map;
    const bool last = static_cast<int>(levels.size()) >= cfg.max_levels;
    if (n <= cfg.coarse_size || last) {
      L.A = std::move(Acur);
      break;
    }
    LevelBuild b = build_level_interp(Acur, cfg.strength_theta, map, &fallback_rows, s);
    if (b.stalled) {
      truncated = true;
      L.A = std::move(Acur);
      break;
    }
    L.A = std::move(Acur);
    L.P = std::move(b.P);
    L.C = std::move(b.C);
    L.F = std::move(b.F);
    L.R = transpose(L.P, s);
    L.pre.bind(cfg.pre, L.A, nullptr, s);
    L.post.bind(cfg.post, L.A, nullptr, s);
    const DCsr AP = spgemm(L.A, L.P, s);
    Acur = spgemm(L.R, AP, s);
    map = std::move(b.coarse_umap);
    L.t.alloc(n, s);
  }
  dense_factor(levels.back().A, coarse, s);
  if (const char* v = std::getenv("MGRX_VERBOSE"); v && v[0] == '1') {
    for (size_t l = 0; l < levels.size(); ++l) {
      const AmgLevelD& L = levels[l];
      std::fprintf(stderr, "[mgrx] amg level %zu: n=%d nnz=%d gs_depth=%d/%d\n", l, L.A.rows, L.A.nnz,
                   L.pre.sched.levels, L.post.sched.levels);
    }
  }
  for (size_t l = 1; l < levels.size(); ++l) {
    const int n = levels[l].A.rows;
    levels[l].r.alloc(n > 0 ? n : 1, s);
    levels[l].z.alloc(n > 0 ? n : 1, s);
  }
}

void AmgHier::vcycle(const double* r, double* z, cudaStream_t s) { vcycle_level(0, r, z, s); }

void AmgHier::vcycle_level(int l, const double* r, double* z, cudaStream_t s) {
  NvtxRange nvtx("mgrx.amg.level", l);
  AmgLevelD& L = levels[l];
  // timing experiment (wrong results): MGRX_VCYCLE_CUT=k replaces the cycle
  // from level k down by z = 0, so the in-situ cost of the levels >= k shows
  // as the difference of two "precond" probes
  static const int cut = [] {
    const char* e = std::getenv("MGRX_VCYCLE_CUT");
    return e ? std::atoi(e) : -1;
  }();
  if (cut >= 0 && l >= cut) {
    MGRX_CK(cudaMemsetAsync(z, 0, sizeof(double) * L.A.rows, s));
    return;
  }
  if (l == ctail) {
    launch_amg_ctail(ctail_desc, ctail_lay, ctail_blob.get(), r, z, s);
    return;
  }
  if (l == tail) {
    launch_amg_tail(tail_desc, tail_blob.get(), r, z, s);
    return;
  }
  if (l == static_cast<int>(levels.size()) - 1) {
    dense_solve(coarse, r, z, s);
    return;
  }
  AmgLevelD& N = levels[l + 1];
  // Jacobi sweep 0 of a pre/post smoother is written by the kernel that
  // produces the smoother's input (restriction / residual) when the level
  // is too large for the folded sweep 0: one launch and one pass fewer.
  const bool pre0 = l > 0 && L.pre.z0_fusable();
  if (pre0) L.pre.jacobi_sweeps(r, nullptr, z, nullptr, s, true);  // z0 from the restriction
  else L.pre.apply(r, nullptr, z, s);                              // z = pre(r)
  spmv_residual(L.A, z, r, nullptr, L.t.get(), s);                 // t = r - A z
  const bool npre0 = l + 1 != tail && l + 1 < static_cast<int>(levels.size()) - 1 && N.pre.z0_fusable();
  if (npre0) spmv_j0(L.R, L.t.get(), N.r.get(), N.pre.dinv.get(), N.pre.spec.weight, N.pre.w2.get(), s);
  else spmv(L.R, L.t.get(), N.r.get(), s);                         // rc = R t
  vcycle_level(l + 1, N.r.get(), N.z.get(), s);                    // ec
  spmv_add(L.P, N.z.get(), z, s);                                  // z += P ec
  if (L.post.z0_fusable()) {
    spmv_residual_j0(L.A, z, r, L.t.get(), L.post.dinv.get(), L.post.spec.weight, L.post.w2.get(), s);
    L.post.jacobi_sweeps(L.t.get(), nullptr, nullptr, z, s, true);  // z += post(t)
  } else {
    spmv_residual(L.A, z, r, nullptr, L.t.get(), s);               // t = r - A z
    L.post.apply_add(L.t.get(), z, s);                             // z += post(t)
  }
}

// ============================================================================
// MGR (proj/src/mgr.cpp:223-326)
// ============================================================================
bool split_prolong_enabled();
void prepare_amg(AmgHier& h, cudaStream_t s);
void prepare_relax(BoundRelax& b, cudaStream_t s) {
  if (b.amg) prepare_amg(*b.amg, s);
}
void prepare_amg(AmgHier& h, cudaStream_t s) {
  for (auto& L : h.levels) {
    for (DCsr* M : {&L.A, &L.P, &L.R}) spmv_prepare(*M, s);
    prepare_relax(L.pre, s);
    prepare_relax(L.post, s);
  }
  h.build_tail(s);
}

TailLevelHost tail_level_host(const AmgLevelD& L);

// Choose the first level (>= 1) from which the rest of the V-cycle fits in
// one CTA's shared memory (Jacobi / l1-Jacobi smoothing, single-block
// coarsest LU) and pack it (MGRX_AMG_TAIL=0: off).
void AmgHier::build_tail(cudaStream_t s) {
  build_single_tail(s);
  // Cluster tail: from the first level of <= kCtMaxRows rows, when that is
  // above the single-CTA tail (MGRX_AMG_CTAIL=0: off).
  ctail = -1;
  // Off by default: bitwise equal (GPU parity suite with MGRX_AMG_CTAIL=1) but
  // measured SLOWER at cfg2 -- levels 4-6 take 91 us in the cluster kernel
  // against 46 us as launches + single-CTA tail (preconditioner 403 -> 457 us;
  // from level 3: 500 us). In-kernel timers: 1.3-3.6 us per published vector
  // (16 x 16 distributed-shared-memory pushes + rendezvous), 3-4.5 us per
  // 857-row product on 16 SMs, 23 us around the one-warp dense solve.
  static const bool con = [] {
    const char* v = std::getenv("MGRX_AMG_CTAIL");
    return v && std::atoi(v) != 0;
  }();
  const int nl = static_cast<int>(levels.size());
  if (!con || nl < 3 || coarse.nb != 1 || coarse.n <= 0 || coarse.n > 256) return;
  auto jac = [](const BoundRelax& b) {
    return (b.spec.kind == Smoother::jacobi || b.spec.kind == Smoother::l1_jacobi) && b.spec.sweeps >= 1;
  };
  for (int t = std::max(1, nl - 1 - kTailMaxLevels); t <= nl - 2; ++t) {
    if (tail >= 0 && t >= tail) return;  // the single-CTA tail already starts here
    static const int max_rows = [] {  // MGRX_CTAIL_MAXROWS: largest level the cluster tail starts at
      const char* v = std::getenv("MGRX_CTAIL_MAXROWS");
      return v ? std::min(std::atoi(v), kCtMaxRows) : kCtMaxRows;
    }();
    if (levels[t].A.rows > max_rows) continue;
    bool ok = true;
    for (int l = t; l < nl - 1 && ok; ++l) ok = jac(levels[l].pre) && jac(levels[l].post);
    if (!ok) continue;
    std::vector<TailLevelHost> lv;
    for (int l = t; l < nl - 1; ++l) lv.push_back(tail_level_host(levels[l]));
    const int nc = coarse.n;
    const std::vector<double> lu = coarse.lu.download(static_cast<size_t>(nc) * nc);
    const std::vector<int> perm = coarse.perm.download(nc);
    std::vector<unsigned char> blob;
    if (!build_ctail_blob(lv, nc, lu, perm, ctail_desc, blob, ctail_lay)) continue;
    ctail_blob.alloc(blob.size(), s);
    ctail_blob.upload(blob.data(), blob.size());
    prepare_amg_ctail(ctail_lay);
    ctail = t;
    if (const char* v = std::getenv("MGRX_VERBOSE"); v && v[0] == '1')
      std::fprintf(stderr, "[mgrx] amg cluster tail from level %d of %d (%d shared bytes per CTA, %zu blob bytes)\n", t,
                   nl, ctail_lay.total, blob.size());
    return;
  }
}

TailLevelHost tail_level_host(const AmgLevelD& L) {
  TailLevelHost h;
  h.m = L.A.rows;
  h.mc = L.R.rows;
  h.a_ptr = L.A.ptr.download(L.A.rows + 1);
  h.a_col = L.A.col.download(L.A.nnz);
  h.a_val = L.A.val.download(L.A.nnz);
  h.r_ptr = L.R.ptr.download(L.R.rows + 1);
  h.r_col = L.R.col.download(L.R.nnz);
  h.r_val = L.R.val.download(L.R.nnz);
  h.p_ptr = L.P.ptr.download(L.P.rows + 1);
  h.p_col = L.P.col.download(L.P.nnz);
  h.p_val = L.P.val.download(L.P.nnz);
  h.dpre = L.pre.dinv.download(L.A.rows);
  h.dpost = L.post.dinv.download(L.A.rows);
  h.pre_sweeps = L.pre.spec.sweeps;
  h.post_sweeps = L.post.spec.sweeps;
  h.pre_w = L.pre.spec.weight;
  h.post_w = L.post.spec.weight;
  return h;
}

void AmgHier::build_single_tail(cudaStream_t s) {
  tail = -1;
  static const bool on = [] {
    const char* v = std::getenv("MGRX_AMG_TAIL");
    return !v || std::atoi(v) != 0;
  }();
  const int nl = static_cast<int>(levels.size());  // levels[nl - 1] is the coarsest
  if (!on || nl < 3 || coarse.nb != 1 || coarse.n <= 0 || coarse.n > 256) return;
  auto jac = [](const BoundRelax& b) {
    return (b.spec.kind == Smoother::jacobi || b.spec.kind == Smoother::l1_jacobi) && b.spec.sweeps >= 1;
  };
  constexpr size_t kBudget = 200 * 1024;
  for (int t = std::max(1, nl - 1 - kTailMaxLevels); t <= nl - 2; ++t) {
    bool ok = true;
    size_t est = 8 * static_cast<size_t>(coarse.n) * coarse.n;
    for (int l = t; l < nl - 1 && ok; ++l) {
      const AmgLevelD& L = levels[l];
      ok = jac(L.pre) && jac(L.post);
      est += 12 * static_cast<size_t>(L.A.nnz + L.R.nnz + L.P.nnz) + 56 * static_cast<size_t>(L.A.rows);
    }
    if (!ok || est > kBudget) continue;
    std::vector<TailLevelHost> lv;
    for (int l = t; l < nl - 1; ++l) {
      const AmgLevelD& L = levels[l];
      TailLevelHost h;
      h.m = L.A.rows;
      h.mc = L.R.rows;
      h.a_ptr = L.A.ptr.download(L.A.rows + 1);
      h.a_col = L.A.col.download(L.A.nnz);
      h.a_val = L.A.val.download(L.A.nnz);
      h.r_ptr = L.R.ptr.download(L.R.rows + 1);
      h.r_col = L.R.col.download(L.R.nnz);
      h.r_val = L.R.val.download(L.R.nnz);
      h.p_ptr = L.P.ptr.download(L.P.rows + 1);
      h.p_col = L.P.col.download(L.P.nnz);
      h.p_val = L.P.val.download(L.P.nnz);
      h.dpre = L.pre.dinv.download(L.A.rows);
      h.dpost = L.post.dinv.download(L.A.rows);
      h.pre_sweeps = L.pre.spec.sweeps;
      h.post_sweeps = L.post.spec.sweeps;
      h.pre_w = L.pre.spec.weight;
      h.post_w = L.post.spec.weight;
      lv.push_back(std::move(h));
    }
    const int nc = coarse.n;
    const std::vector<double> lu = coarse.lu.download(static_cast<size_t>(nc) * nc);
    const std::vector<int> perm = coarse.perm.download(nc);
    std::vector<unsigned char> blob;
    if (!build_tail_blob(lv, nc, lu, perm, kBudget, tail_desc, blob)) continue;
    tail_blob.alloc(blob.size(), s);
    tail_blob.upload(blob.data(), blob.size());
    prepare_amg_tail(tail_desc);
    tail = t;
    if (const char* v = std::getenv("MGRX_VERBOSE"); v && v[0] == '1')
      std::fprintf(stderr, "[mgrx] amg tail from level %d of %d (%d shared bytes)\n", t, nl, tail_desc.total_bytes);
    return;
  }
}

void MgrHier::setup(const DCsr& A, const std::vector<int>& labels, const std::vector<std::string>& fields,
                    const std::vector<int>* umap_in, const Strategy& strat, cudaStream_t s) {
  NvtxRange nvtx("mgrx.mgr_setup");
  if (A.rows != A.cols) throw InvalidArgument("mgr_setup: matrix must be square");
  if (static_cast<int>(labels.size()) != A.rows)
    throw InvalidArgument("mgr_setup: partition size does not match the matrix");
  if (umap_in && static_cast<int>(umap_in->size()) != A.rows)
    throw InvalidArgument("mgr_setup: unknown_map size mismatch");
  auto field_id = [&](const std::string& name) {
    for (size_t k = 0; k < fields.size(); ++k)
      if (fields[k] == name) return static_cast<int>(k);
    throw InvalidArgument("unknown field name: " + name);
  };
  {
    std::unordered_set<std::string> used;
    for (const auto& lv : strat.levels) {
      if (lv.f_fields.empty()) throw InvalidArgument("mgr_setup: a level with no f_fields");
      for (const auto& f : lv.f_fields) {
        field_id(f);
        if (!used.insert(f).second) throw InvalidArgument("mgr_setup: field eliminated twice: " + f);
      }
    }
  }
  if (strat.coarse.kind == Coarse::gmres_inner)
    throw RuntimeError("coarse solver gmres_inner is not supported on the device path");
  n = A.rows;
  coarse_spec = strat.coarse;
  levels.clear();
  DCsr Acur = csr_copy(A, s);  // level operator handed to each level in turn
  DVec<int> lab(n > 0 ? n : 1, s);
  lab.upload(labels.data(), n);
  std::vector<int> umap;
  if (umap_in) umap = *umap_in;

  for (const auto& spec : strat.levels) {
    levels.emplace_back();
    NvtxRange nvtx_level("mgrx.mgr_setup.level", static_cast<int>(levels.size()) - 1);
    MgrLevelD& L = levels.back();
    L.A = std::move(Acur);
    const int nl = L.A.rows;
    // split_ids (mgr.cpp:27-44)
    std::vector<uint8_t> mask(fields.size(), 0);
    for (const auto& f : spec.f_fields) mask[field_id(f)] = 1;
    DVec<uint8_t> dmask(mask.size(), s), isf(nl > 0 ? nl : 1, s), isc(nl > 0 ? nl : 1, s);
    dmask.upload(mask.data(), mask.size());
    launch1d(k_split, nl, s, lab.get(), dmask.get(), isf.get(), isc.get());
    const int nf = select_flagged(isf.get(), nl, L.F, s);
    if (nf == 0) throw InvalidArgument("split: F set is empty");
    const int nc = select_flagged(isc.get(), nl, L.C, s);
    if (nc == 0) throw InvalidArgument("split: C set is empty (all fields eliminated)");
    DVec<int> cpos;
    rank_flags(isf.get(), nl, L.fpos, s);
    rank_flags(isc.get(), nl, cpos, s);

    L.Aff = extract(L.A, L.F.get(), nf, L.F.get(), nf, s);
    // Diagonal A_FF (jacobi transfers, or ideal with a structurally diagonal
    // A_FF): W = dinv_F * A_FC in the interpolation / restriction kernels.
    // Otherwise ideal transfers solve with the declared block layout or a
    // dense LU (ff_inverse_times).
    const bool ideal_any = spec.interp == Interp::ideal || spec.restrict_kind == Restrict::ideal;
    const bool diag_ff = ideal_any ? structurally_diagonal(L.Aff, s) : true;
    DVec<double> dinv_f;
    bool have_dinv = false;
    auto need_dinv = [&] {
      if (!have_dinv) diag_inverse(L.Aff, dinv_f, s);
      have_dinv = true;
    };

    // P (build_interp)
    if (spec.interp == Interp::jacobi || diag_ff) {
      need_dinv();
      DVec<int> cnt(nl, s);
      L.P.rows = nl;
      L.P.cols = nc;
      L.P.ptr.alloc(nl + 1, s);
      launch1d(k_mgr_interp<false>, nl, s, L.A.ptr.get(), L.A.col.get(), L.A.val.get(), L.fpos.get(),
               cpos.get(), dinv_f.get(), cnt.get(), static_cast<const int*>(nullptr),
               static_cast<int*>(nullptr), static_cast<double*>(nullptr));
      L.P.nnz = static_cast<int>(exclusive_scan(cnt.get(), L.P.ptr.get(), nl, s));
      L.P.col.alloc(L.P.nnz, s);
      L.P.val.alloc(L.P.nnz, s);
      launch1d(k_mgr_interp<true>, nl, s, L.A.ptr.get(), L.A.col.get(), L.A.val.get(), L.fpos.get(),
               cpos.get(), dinv_f.get(), static_cast<int*>(nullptr), L.P.ptr.get(), L.P.col.get(),
               L.P.val.get());
    } else {
      const DCsr Afc = extract(L.A, L.F.get(), nf, L.C.get(), nc, s);
      const DCsr W = ff_solve(L.Aff, Afc, spec.ff_block_sizes, s);
      DVec<int> cnt(nl, s);
      L.P.rows = nl;
      L.P.cols = nc;
      L.P.ptr.alloc(nl + 1, s);
      launch1d(k_interp_from_w<false>, nl, s, L.fpos.get(), cpos.get(), W.ptr.get(), W.col.get(), W.val.get(),
               cnt.get(), static_cast<const int*>(nullptr), static_cast<int*>(nullptr),
               static_cast<double*>(nullptr));
      L.P.nnz = static_cast<int>(exclusive_scan(cnt.get(), L.P.ptr.get(), nl, s));
      L.P.col.alloc(L.P.nnz, s);
      L.P.val.alloc(L.P.nnz, s);
      launch1d(k_interp_from_w<true>, nl, s, L.fpos.get(), cpos.get(), W.ptr.get(), W.col.get(), W.val.get(),
               static_cast<int*>(nullptr), L.P.ptr.get(), L.P.col.get(), L.P.val.get());
    }
    // R (build_restrict)
    L.injection = spec.restrict_kind == Restrict::injection;
    if (L.injection || spec.restrict_kind == Restrict::jacobi || diag_ff) {
      if (!L.injection) need_dinv();
      DVec<int> cnt(nc, s);
      L.R.rows = nc;
      L.R.cols = nl;
      L.R.ptr.alloc(nc + 1, s);
      launch1d(k_mgr_restrict<false>, nc, s, L.injection, L.A.ptr.get(), L.A.col.get(), L.A.val.get(),
               L.C.get(), L.fpos.get(), static_cast<const double*>(dinv_f.get()), cnt.get(),
               static_cast<const int*>(nullptr), static_cast<int*>(nullptr), static_cast<double*>(nullptr));
      L.R.nnz = static_cast<int>(exclusive_scan(cnt.get(), L.R.ptr.get(), nc, s));
      L.R.col.alloc(L.R.nnz, s);
      L.R.val.alloc(L.R.nnz, s);
      launch1d(k_mgr_restrict<true>, nc, s, L.injection, L.A.ptr.get(), L.A.col.get(), L.A.val.get(),
               L.C.get(), L.fpos.get(), static_cast<const double*>(dinv_f.get()), static_cast<int*>(nullptr),
               L.R.ptr.get(), L.R.col.get(), L.R.val.get());
    } else {
      // A_CF A_FF^{-1} = (A_FF^{-T} A_CF^T)^T (proj/src/mgr.cpp:128-133)
      const DCsr Acf = extract(L.A, L.C.get(), nc, L.F.get(), nf, s);
      const DCsr AffT = transpose(L.Aff, s);
      const DCsr AcfT = transpose(Acf, s);
      const DCsr Zt = ff_solve(AffT, AcfT, spec.ff_block_sizes, s);
      const DCsr Z = transpose(Zt, s);
      DVec<int> cnt(nc, s);
      L.R.rows = nc;
      L.R.cols = nl;
      L.R.ptr.alloc(nc + 1, s);
      launch1d(k_restrict_from_z<false>, nc, s, L.C.get(), L.F.get(), Z.ptr.get(), Z.col.get(), Z.val.get(),
               cnt.get(), static_cast<const int*>(nullptr), static_cast<int*>(nullptr),
               static_cast<double*>(nullptr));
      L.R.nnz = static_cast<int>(exclusive_scan(cnt.get(), L.R.ptr.get(), nc, s));
      L.R.col.alloc(L.R.nnz, s);
      L.R.val.alloc(L.R.nnz, s);
      launch1d(k_restrict_from_z<true>, nc, s, L.C.get(), L.F.get(), Z.ptr.get(), Z.col.get(), Z.val.get(),
               static_cast<int*>(nullptr), L.R.ptr.get(), L.R.col.get(), L.R.val.get());
    }
    // F-relaxation smoother on A_FF (+ optional global relaxation on A)
    std::vector<int> umap_f;
    if (!umap.empty()) umap_f = gather_host(umap, L.F.download(nf));
    L.f_relax.bind(spec.f_relax, L.Aff, umap.empty() ? nullptr : &umap_f, s);
    if (spec.global_relax) {
      L.g_relax.emplace();
      L.g_relax->bind(*spec.global_relax, L.A, umap.empty() ? nullptr : &umap, s);
    }
    // Galerkin coarse operator R (A P) (mgr.cpp:148-152). With injection,
    // R(AP) is rows C of AP: every product is AP(C_j, c) * 1.0, exact.
    {
      const DCsr AP = spgemm(L.A, L.P, s);
      DCsr Anext = L.injection ? gather_rows(AP, L.C.get(), nc, s) : spgemm(L.R, AP, s);
      if (L.injection && !spec.global_relax) L.Acf = extract(L.A, L.C.get(), nc, L.F.get(), nf, s);
      Acur = std::move(Anext);
    }
    // carry labels / unknown map to the C dofs
    {
      DVec<int> lab2(nc, s);
      launch1d(k_gather_int, nc, s, L.C.get(), lab.get(), lab2.get());
      lab = std::move(lab2);
      if (!umap.empty()) umap = gather_host(umap, L.C.download(nc));
    }
    L.zF.alloc(nf, s);
    L.rc.alloc(nc, s);
    L.e.alloc(nc, s);
    L.t.alloc(nl, s);
    L.zfull.alloc(nl, s);
  }
  A_coarse = std::move(Acur);
  switch (strat.coarse.kind) {
    case Coarse::dense_lu:
      dense_factor(A_coarse, coarse_lu, s);
      break;
    case Coarse::amg_vcycle: {
      std::vector<int> um;
      if (strat.coarse.use_unknown_map) {
        if (umap.empty())
          throw InvalidArgument("mgr_setup: coarse solver requests an unknown map, none given");
        um = umap;
      }
      coarse_amg = std::make_unique<AmgHier>();
      coarse_amg->setup(A_coarse, strat.coarse.amg, um, s);
      break;
    }
    case Coarse::gmres_inner:
      break;
  }
  const int ncs = A_coarse.rows > 0 ? A_coarse.rows : 1;
  ct.alloc(ncs, s);
  cd.alloc(ncs, s);
  // block plans of the staged SpMV for every solve-path matrix
  for (auto& L : levels) {
    for (DCsr* M : {&L.A, &L.P, &L.R, &L.Acf, &L.Aff}) spmv_prepare(*M, s);
    if (L.injection && !L.g_relax && split_prolong_enabled())
      prolong_prepare(L.P, L.F.get(), static_cast<int>(L.F.size()), L.C.get(), static_cast<int>(L.C.size()), L.pplan,
                      s);
    prepare_relax(L.f_relax, s);
    if (L.g_relax) prepare_relax(*L.g_relax, s);
  }
  spmv_prepare(A_coarse, s);
  if (coarse_amg) prepare_amg(*coarse_amg, s);
}

void MgrHier::coarse_solve(const double* v, double* z, cudaStream_t s) {
  if (coarse_spec.kind == Coarse::dense_lu) {
    dense_solve(coarse_lu, v, z, s, exact_dense_);
    return;
  }
  // z = V(v); z += V(v - A_c z) for the remaining cycles (mgr.cpp:181-186)
  coarse_amg->vcycle(v, z, s);
  for (int c = 1; c < coarse_spec.cycles; ++c) {
    spmv_residual(A_coarse, z, v, nullptr, ct.get(), s);
    coarse_amg->vcycle(ct.get(), cd.get(), s);
    vec_add(A_coarse.rows, cd.get(), z, s);
  }
}

void MgrHier::apply(const double* v, double* z, cudaStream_t s, bool exact) {
  TeamSums team_sums(!exact, exact);  // exact: bitwise kernels whatever the caller's scope
  exact_dense_ = exact;
  apply_level(0, v, z, s);
  exact_dense_ = true;
}

bool split_prolong_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("MGRX_SPLIT_PROLONG");
    return !(e && e[0] == '0');
  }();
  return on;
}

void MgrHier::prolong(int l, const double* e, const double* zF, double* z, cudaStream_t s) {
  MgrLevelD& L = levels[l];
  if (L.pplan.w > 0) spmv_prolong_split(L.pplan, e, zF, z, s);
  else spmv_prolong(L.P, e, L.fpos.get(), zF, z, s);
}

void MgrHier::apply_graph(const double* v, double* z, cudaStream_t s, bool exact) {
  static const bool enabled = [] {
    const char* e = std::getenv("MGRX_GRAPHS");
    return !(e && e[0] == '0');
  }();
  if (!enabled) {
    apply(v, z, s, exact);
    return;
  }
  auto it = graphs_.find({v, z, exact});
  if (it == graphs_.end()) {
    Captured c;
    const long long l0 = g_launches;
    cudaGraph_t g;
    MGRX_CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    try {
      apply(v, z, s, exact);
    } catch (...) {
      cudaStreamEndCapture(s, &g);
      throw;
    }
    MGRX_CK(cudaStreamEndCapture(s, &g));
    MGRX_CK(cudaGraphInstantiate(&c.exec, g, 0));
    MGRX_CK(cudaGraphDestroy(g));
    c.nodes = g_launches - l0;
    g_launches = l0;
    it = graphs_.emplace(std::make_tuple(v, z, exact), c).first;
  }
  MGRX_CK(cudaGraphLaunch(it->second.exec, s));
  count_launch(it->second.nodes);
}

void MgrHier::tune_spmv(cudaStream_t s) {
  static const bool on = [] {
    const char* e = std::getenv("MGRX_TUNE_INSITU");
    return !e || std::atoi(e) != 0;
  }();
  if (!on || n == 0) return;
  const char* pf = std::getenv("MGRX_SPMV_PLAN_FILE");
  std::vector<DCsr*> cands;
  auto add = [&](DCsr& M) {
    if (M.xt_plan_nblk > 0) cands.push_back(&M);
  };
  std::function<void(AmgHier*)> add_amg = [&](AmgHier* a) {
    if (!a) return;
    for (auto& L : a->levels) {
      add(L.A);
      add(L.P);
      add(L.R);
    }
  };
  for (auto& L : levels) {
    for (DCsr* M : {&L.A, &L.P, &L.R, &L.Acf, &L.Aff}) add(*M);
    add_amg(L.f_relax.amg.get());
    if (L.g_relax) add_amg(L.g_relax->amg.get());
  }
  add(A_coarse);
  add_amg(coarse_amg.get());
  if (cands.empty()) return;
  std::stable_sort(cands.begin(), cands.end(), [](const DCsr* a, const DCsr* b) { return a->nnz > b->nnz; });
  // decisions recorded by an earlier run (so that a profiler sees the production choices)
  if (pf)
    if (FILE* f = std::fopen(pf, "r")) {
      // (the xt_on / xt_off lines are in candidate order: operators of equal
      // size, e.g. the coarse system and its copy as AMG level 0, stay apart)
      std::vector<int> dec(cands.size(), -1);
      int r, c, z;
      char what[16];
      size_t i = 0;
      while (std::fscanf(f, "%d %d %d %15s", &r, &c, &z, what) == 4) {
        const bool on_line = !std::strcmp(what, "xt_on"), off_line = !std::strcmp(what, "xt_off");
        if (!on_line && !off_line) continue;
        if (i < cands.size() && r == cands[i]->rows && c == cands[i]->cols && z == cands[i]->nnz)
          dec[i] = on_line ? 1 : 0;
        ++i;
      }
      std::fclose(f);
      if (std::find(dec.begin(), dec.end(), -1) == dec.end()) {
        for (size_t i = 0; i < cands.size(); ++i) {
          cands[i]->xt_nblk = dec[i] ? cands[i]->xt_plan_nblk : 0;
          if (!dec[i]) spmv_drop_xtile(*cands[i]);
        }
        return;
      }
    }
  DVec<double> v(n, s), z(n, s);
  v.zero();
  cudaEvent_t e0, e1;
  MGRX_CK(cudaEventCreate(&e0));
  MGRX_CK(cudaEventCreate(&e1));
  const long long l0 = g_launches;
  int reps = 3;
  auto time = [&] {
    float best = 1e30f;
    for (int rep = 0; rep < reps; ++rep) {
      MGRX_CK(cudaEventRecord(e0, s));
      apply(v.get(), z.get(), s, false);
      MGRX_CK(cudaEventRecord(e1, s));
      MGRX_CK(cudaEventSynchronize(e1));
      float ms = 0.f;
      MGRX_CK(cudaEventElapsedTime(&ms, e0, e1));
      best = std::min(best, ms);
    }
    return best;
  };
  apply(v.get(), z.get(), s, false);  // warm
  float cur = time();
  // (sweep-bound strategies, e.g. exact Gauss-Seidel: one repetition, or no
  // pass at all when an application takes tens of milliseconds)
  if (cur > 5.f) reps = 1;
  if (cur > 30.f) cands.clear();
  const bool verbose = [] {
    const char* e = std::getenv("MGRX_VERBOSE");
    return e && e[0] == '1';
  }();
  std::vector<DCsr*> team_off;
  for (DCsr* M : cands) {
    if (M->vec > 0 || M->tb > 0) {
      // the application runs this operator through a team-sum kernel
      // (tolerance mode), so the window's switch would not show: time the
      // window against the team kernel instead, and keep the window for the
      // bitwise paths either way
      const int vec0 = M->vec, tb0 = M->tb;
      M->vec = 0;
      M->tb = 0;
      M->xt_nblk = M->xt_plan_nblk;
      const float t = time();
      if (verbose)
        std::fprintf(stderr, "tune_spmv rows %d nnz %d: team sums %.1f us, x-window %.1f us\n", M->rows, M->nnz,
                     1e3f * cur, 1e3f * t);
      if (t < 0.995f * cur) {
        cur = t;
        team_off.push_back(M);
      } else {
        M->vec = vec0;
        M->tb = tb0;
      }
      continue;
    }
    const int was = M->xt_nblk;
    M->xt_nblk = was ? 0 : M->xt_plan_nblk;
    const float t = time();
    if (verbose)
      std::fprintf(stderr, "tune_spmv rows %d nnz %d: x-window %s %.1f us, %s %.1f us\n", M->rows, M->nnz,
                   was ? "on" : "off", 1e3f * cur, was ? "off" : "on", 1e3f * t);
    if (t < 0.995f * cur) cur = t;
    else M->xt_nblk = was;
  }
  if (pf)
    if (FILE* f = std::fopen(pf, "a")) {
      for (DCsr* M : cands) std::fprintf(f, "%d %d %d %s\n", M->rows, M->cols, M->nnz, M->xt_nblk ? "xt_on" : "xt_off");
      // (later lines win in vec_try / tbsr_try's replay)
      for (DCsr* M : team_off) std::fprintf(f, "%d %d %d novec\n%d %d %d notbsr\n", M->rows, M->cols, M->nnz, M->rows, M->cols, M->nnz);
      std::fclose(f);
    }
  for (DCsr* M : cands)
    if (M->xt_nblk == 0) spmv_drop_xtile(*M);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  g_launches = l0;
  check(s);
}

MgrHier::~MgrHier() {
  for (auto& kv : graphs_)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
}

void MgrHier::corrupt_transfer(int l, double factor, cudaStream_t s) {
  if (l < 0 || l >= static_cast<int>(levels.size()))
    throw InvalidArgument("corrupt_transfer: no MGR level " + std::to_string(l));
  MgrLevelD& L = levels[l];
  if (L.P.nnz > 0) vec_scale(L.P.nnz, L.P.val.get(), factor, L.P.val.get(), s);
  // plans that carry their own copy of the values would keep the clean P
  L.P.bsr = 0;
  L.P.nslice = 0;
  L.P.tb = 0;
  L.pplan.w = 0;
  MGRX_CK(cudaStreamSynchronize(s));
  for (auto& kv : graphs_)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  graphs_.clear();
}

void MgrHier::apply_level(int l, const double* v, double* z, cudaStream_t s) {
  if (l == static_cast<int>(levels.size())) {
    NvtxRange nvtx("mgrx.mgr.coarse_solve");
    coarse_solve(v, z, s);
    return;
  }
  NvtxRange nvtx("mgrx.mgr.level", l);
  MgrLevelD& L = levels[l];
  const int nf = static_cast<int>(L.F.size()), nc = static_cast<int>(L.C.size());
  if (L.injection && !L.g_relax) {
    // Fast path, arithmetic identical to mgr.cpp:206-217 with z = 0 on C:
    //   zF = f_relax(v_F)
    //   rc = v_C - A_CF zF      (R is injection; A_CC z_C contributes exact zeros)
    //   e  = next level(rc)
    //   z  = [0 + zF ; 0] + P e  (one fused prolongation kernel)
    L.f_relax.apply(v, L.F.get(), L.zF.get(), s);
    spmv_residual(L.Acf, L.zF.get(), v, L.C.get(), L.rc.get(), s);
    apply_level(l + 1, L.rc.get(), L.e.get(), s);
    prolong(l, L.e.get(), L.zF.get(), z, s);
    (void)nf;
    (void)nc;
    return;
  }
  // General path (global relaxation and/or non-injection restriction).
  const int nl = L.A.rows;
  const double* r = v;
  if (L.g_relax) {
    L.g_relax->apply(v, nullptr, z, s);
    spmv_residual(L.A, z, v, nullptr, L.t.get(), s);
    r = L.t.get();
  } else {
    MGRX_CK(cudaMemsetAsync(z, 0, sizeof(double) * nl, s));
  }
  L.f_relax.apply(r, L.F.get(), L.zF.get(), s);
  launch1d(k_scatter_add, nf, s, L.F.get(), L.zF.get(), z);
  spmv_residual(L.A, z, v, nullptr, L.t.get(), s);
  spmv(L.R, L.t.get(), L.rc.get(), s);
  apply_level(l + 1, L.rc.get(), L.e.get(), s);
  spmv_add(L.P, L.e.get(), z, s);
}

void MgrHier::check(cudaStream_t s) {
  for (auto& L : levels) {
    L.f_relax.check(s);
    if (L.g_relax) L.g_relax->check(s);
  }
  if (coarse_amg)
    for (auto& L : coarse_amg->levels) {
      L.pre.check(s);
      L.post.check(s);
    }
}

}  // namespace mgrx
