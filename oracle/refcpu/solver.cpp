// refcpu — CPU ORACLE (test infrastructure only; see csr.hpp header).
// Restates proj/src/{relax,amg,krylov,mgr}.cpp without Eigen. Each function
// cites the reference lines whose behaviour it reproduces.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <unordered_set>

#include "solver.hpp"

namespace refcpu {

// ============================================================================
// relax — proj/src/relax.cpp
// ============================================================================
namespace {

Partition tile_check(const Partition& p, Index n) {  // relax.cpp:12-23
  if (p.empty()) return {{0, n}};
  Index expect = 0;
  for (const auto& [b, e] : p) {
    if (b != expect || e <= b)
      throw std::invalid_argument("smoother partition ranges must tile [0,n) in order");
    expect = e;
  }
  if (expect != n) throw std::invalid_argument("smoother partition does not cover the matrix");
  return p;
}

std::vector<Index> owners(const Partition& p, Index n) {  // relax.cpp:26-31
  std::vector<Index> o(n);
  for (Index r = 0; r < static_cast<Index>(p.size()); ++r)
    for (Index i = p[r].first; i < p[r].second; ++i) o[i] = r;
  return o;
}

}  // namespace

Vec l1_diagonal(const Csr& A, const Partition& partition) {
  const Index n = A.rows;
  const Partition p = tile_check(partition, n);
  const std::vector<Index> o = owners(p, n);
  Vec d(n, 0.0);
  for (Index i = 0; i < n; ++i)
    for (Index k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
      const Index j = A.col[k];
      if (j == i)
        d[i] += A.val[k];
      else if (o[j] != o[i])
        d[i] += std::abs(A.val[k]);
    }
  return d;
}

void jacobi_sweep(const Csr& A, const Vec& b, Vec& x, Real weight) {
  const Vec dinv = diag_inverse(A);
  const Vec r = sub(b, spmv(A, x));
  for (size_t i = 0; i < x.size(); ++i) x[i] += weight * (dinv[i] * r[i]);
}

void hybrid_l1_gs_sweep(const Csr& A, const Vec& l1d, const Vec& b, Vec& x, bool forward,
                        const Partition& partition) {
  const Index n = A.rows;
  if (static_cast<Index>(b.size()) != n || static_cast<Index>(x.size()) != n ||
      static_cast<Index>(l1d.size()) != n)
    throw std::invalid_argument("hybrid_l1_gs_sweep: size mismatch");
  const Partition p = tile_check(partition, n);
  const std::vector<Index> o = owners(p, n);
  const Vec snap = x;
  for (Index i = 0; i < n; ++i)
    if (l1d[i] == 0.0)
      throw std::runtime_error("hybrid_l1_gs_sweep: zero L1 diagonal at row " + std::to_string(i));
  for (const auto& [lo, hi] : p) {
    for (Index s = 0; s < hi - lo; ++s) {
      const Index i = forward ? lo + s : hi - 1 - s;
      Real acc = b[i];
      for (Index k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
        const Index j = A.col[k];
        acc -= A.val[k] * (o[j] == o[i] ? x[j] : snap[j]);
      }
      x[i] += acc / l1d[i];
    }
  }
}

void hybrid_l1_gs_sweep(const Csr& A, const Vec& b, Vec& x, bool forward, const Partition& p) {
  hybrid_l1_gs_sweep(A, l1_diagonal(A, p), b, x, forward, p);
}

BoundSmoother BoundSmoother::bind(const SmootherSpec& spec, const Csr& A,
                                  const std::vector<int>* unknown_map) {
  if (A.rows != A.cols) throw std::invalid_argument("smoother: matrix must be square");
  if (spec.sweeps < 1) throw std::invalid_argument("smoother: sweeps must be >= 1");
  if (!(spec.weight > 0.0 && spec.weight < 2.0))
    throw std::invalid_argument("smoother: weight must lie in (0, 2)");
  BoundSmoother s;
  s.spec_ = spec;
  s.A_ = std::make_shared<const Csr>(A);
  const Index n = A.rows;
  switch (spec.kind) {
    case SmootherKind::jacobi:
      s.dinv_ = diag_inverse(A);
      break;
    case SmootherKind::l1_jacobi: {
      Partition singles(n);
      for (Index i = 0; i < n; ++i) singles[i] = {i, i + 1};
      const Vec d = l1_diagonal(A, singles);
      s.dinv_.resize(n);
      for (Index i = 0; i < n; ++i) {
        if (d[i] == 0.0) throw std::runtime_error("smoother: zero L1 diagonal at row " + std::to_string(i));
        s.dinv_[i] = 1.0 / d[i];
      }
      break;
    }
    case SmootherKind::hybrid_l1_gs_forward:
    case SmootherKind::hybrid_l1_gs_backward:
      s.partition_ = tile_check(spec.partition, n);
      s.l1d_ = l1_diagonal(A, s.partition_);
      for (Index i = 0; i < n; ++i)
        if (s.l1d_[i] == 0.0) throw std::runtime_error("smoother: zero L1 diagonal at row " + std::to_string(i));
      break;
    case SmootherKind::block_jacobi_exact:
      if (spec.block_sizes.empty())
        throw std::invalid_argument("smoother: block_jacobi_exact requires block sizes");
      s.block_lu_ = std::make_shared<BlockDiagonalLU>(A, BlockLayout::from_sizes(spec.block_sizes));
      break;
    case SmootherKind::dense_lu:
      s.dense_lu_ = std::make_shared<DenseLU>(factor_dense(A));
      break;
    case SmootherKind::amg_vcycle: {
      AmgConfig cfg = spec.amg ? *spec.amg : AmgConfig{};
      if (spec.use_unknown_map) {
        if (unknown_map == nullptr)
          throw std::invalid_argument("smoother: use_unknown_map set but no unknown map supplied");
        cfg.unknown_map = *unknown_map;
      }
      s.amg_ = std::make_shared<AmgHierarchy>(amg_setup(A, cfg));
      break;
    }
  }
  return s;
}

Vec BoundSmoother::apply(const Vec& r) const {
  if (!A_) throw std::logic_error("smoother: apply before bind");
  const Csr& A = *A_;
  if (static_cast<Index>(r.size()) != A.rows)
    throw std::invalid_argument("smoother: residual size mismatch");
  if (spec_.kind == SmootherKind::dense_lu) return dense_lu_->solve(r);
  if (spec_.kind == SmootherKind::block_jacobi_exact) return block_lu_->solve(r);
  const Index n = A.rows;
  const Real w = spec_.weight;
  Vec z(n, 0.0);
  for (Index sweep = 0; sweep < spec_.sweeps; ++sweep) {
    switch (spec_.kind) {
      case SmootherKind::jacobi:
      case SmootherKind::l1_jacobi:
        if (sweep == 0) {
          for (Index i = 0; i < n; ++i) z[i] = w * (dinv_[i] * r[i]);
        } else {
          const Vec d = sub(r, spmv(A, z));
          for (Index i = 0; i < n; ++i) z[i] += w * (dinv_[i] * d[i]);
        }
        break;
      case SmootherKind::hybrid_l1_gs_forward:
        hybrid_l1_gs_sweep(A, l1d_, r, z, true, partition_);
        break;
      case SmootherKind::hybrid_l1_gs_backward:
        hybrid_l1_gs_sweep(A, l1d_, r, z, false, partition_);
        break;
      case SmootherKind::amg_vcycle:
        if (sweep == 0) {
          z = amg_vcycle(*amg_, r);
        } else {
          const Vec c = amg_vcycle(*amg_, sub(r, spmv(A, z)));
          for (Index i = 0; i < n; ++i) z[i] += c[i];
        }
        break;
      default:
        break;
    }
  }
  return z;
}

// ============================================================================
// amg — proj/src/amg.cpp
// ============================================================================
Csr strength_graph(const Csr& A, Real theta) {  // amg.cpp:11-34
  if (A.rows != A.cols) throw std::invalid_argument("strength_graph: matrix must be square");
  std::vector<Triplet> e;
  for (Index i = 0; i < A.rows; ++i) {
    Real mneg = 0.0, mabs = 0.0;
    for (Index k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
      if (A.col[k] == i) continue;
      mneg = std::max(mneg, -A.val[k]);
      mabs = std::max(mabs, std::abs(A.val[k]));
    }
    if (mabs == 0.0) continue;
    const bool neg = mneg > 0.0;
    const Real cut = theta * (neg ? mneg : mabs);
    for (Index k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
      if (A.col[k] == i) continue;
      const Real m = neg ? -A.val[k] : std::abs(A.val[k]);
      if (m >= cut && m > 0.0) e.push_back({i, A.col[k], 1.0});
    }
  }
  return from_triplets(A.rows, A.rows, e);
}

void pmis_coarsen(const Csr& S, IndexList& C, IndexList& F) {  // amg.cpp:36-86
  const Index n = S.rows;
  C.clear();
  F.clear();
  std::vector<Index> lam(n, 0);
  for (Index k = 0; k < S.ptr[n]; ++k) ++lam[S.col[k]];
  const Csr St = transpose(S);
  enum : unsigned char { kU = 0, kC = 1, kF = 2 };
  std::vector<unsigned char> st(n, kU);
  Index remaining = n;
  auto neighbours = [&](Index i, auto&& fn) {
    for (Index k = S.ptr[i]; k < S.ptr[i + 1]; ++k) fn(S.col[k]);
    for (Index k = St.ptr[i]; k < St.ptr[i + 1]; ++k) fn(St.col[k]);
  };
  std::vector<Index> win;
  while (remaining > 0) {
    win.clear();
    for (Index i = 0; i < n; ++i) {
      if (st[i] != kU) continue;
      bool ok = true;
      neighbours(i, [&](Index j) {
        if (!ok || j == i || st[j] != kU) return;
        if (!(lam[i] > lam[j] || (lam[i] == lam[j] && i < j))) ok = false;
      });
      if (ok) win.push_back(i);
    }
    if (win.empty()) throw std::logic_error("pmis_coarsen: stalled selection round");
    for (Index i : win) {
      st[i] = kC;
      --remaining;
    }
    for (Index i : win)
      neighbours(i, [&](Index j) {
        if (st[j] == kU) {
          st[j] = kF;
          --remaining;
        }
      });
  }
  for (Index i = 0; i < n; ++i) (st[i] == kC ? C : F).push_back(i);
}

Csr classical_interp(const Csr& A, const Csr& S, const IndexList& C, const IndexList& F,
                     Index* fallback_rows) {  // amg.cpp:88-141
  const Index n = A.rows;
  if (static_cast<Index>(C.size() + F.size()) != n)
    throw std::invalid_argument("classical_interp: C/F do not partition the dofs");
  std::vector<Index> cid(n, -1);
  for (Index k = 0; k < static_cast<Index>(C.size()); ++k) cid[C[k]] = k;
  Index fb = 0;
  std::vector<Triplet> e;
  for (Index c : C) e.push_back({c, cid[c], 1.0});
  std::vector<char> strong(n, 0);
  for (Index i : F) {
    for (Index k = S.ptr[i]; k < S.ptr[i + 1]; ++k) strong[S.col[k]] = 1;
    Real aii = 0.0, rsum = 0.0, csum = 0.0, rmax = 0.0;
    for (Index k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
      const Index j = A.col[k];
      rmax = std::max(rmax, std::abs(A.val[k]));
      if (j == i) {
        aii = A.val[k];
        continue;
      }
      rsum += A.val[k];
      if (cid[j] >= 0 && strong[j]) csum += A.val[k];
    }
    if (aii == 0.0) throw std::runtime_error("classical_interp: zero diagonal at an F-row");
    if (std::abs(csum) > 1e-14 * rmax) {
      const Real scale = rsum / (aii * csum);
      for (Index k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
        const Index j = A.col[k];
        if (j == i || cid[j] < 0 || !strong[j]) continue;
        e.push_back({i, cid[j], -A.val[k] * scale});
      }
    } else {
      ++fb;
      for (Index k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
        const Index j = A.col[k];
        if (j == i || cid[j] < 0) continue;
        e.push_back({i, cid[j], -A.val[k] / aii});
      }
    }
    for (Index k = S.ptr[i]; k < S.ptr[i + 1]; ++k) strong[S.col[k]] = 0;
  }
  if (fallback_rows) *fallback_rows += fb;
  return from_triplets(n, static_cast<Index>(C.size()), e);
}

namespace {

struct LevelInterp {
  Csr P;
  std::vector<int> coarse_unknowns;
  IndexList C, F;  // global splitting at this level
  bool stalled = false;
};

// amg.cpp:147-230: scalar or per-unknown coarsening; coarse order follows the
// fine order (rank of each C point among all C points).
LevelInterp level_interp(const Csr& A, const AmgConfig& cfg, const std::vector<int>& umap,
                         Index* fallback_rows) {
  const Index n = A.rows;
  LevelInterp out;
  std::vector<char> is_c(n, 0);
  std::vector<Triplet> local;  // (global row, group-local coarse col, value)
  std::vector<std::pair<IndexList, size_t>> groups;  // (idx, first triplet)
  std::vector<IndexList> group_c;
  std::vector<size_t> group_end;

  auto run_group = [&](const Csr& Asub, const IndexList& idx) {
    IndexList Cs, Fs;
    const Csr S = strength_graph(Asub, cfg.strength_theta);
    pmis_coarsen(S, Cs, Fs);
    const Csr P = classical_interp(Asub, S, Cs, Fs, fallback_rows);
    const size_t first = local.size();
    for (Index r = 0; r < P.rows; ++r)
      for (Index k = P.ptr[r]; k < P.ptr[r + 1]; ++k) local.push_back({idx[r], P.col[k], P.val[k]});
    IndexList cg(Cs.size());
    for (size_t k = 0; k < Cs.size(); ++k) {
      cg[k] = idx[Cs[k]];
      is_c[cg[k]] = 1;
    }
    groups.push_back({idx, first});
    group_c.push_back(cg);
    group_end.push_back(local.size());
  };

  if (umap.empty()) {
    IndexList all(n);
    std::iota(all.begin(), all.end(), 0);
    run_group(A, all);
  } else {
    std::vector<int> ids = umap;
    std::sort(ids.begin(), ids.end());
    ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
    for (int id : ids) {
      IndexList idx;
      for (Index i = 0; i < n; ++i)
        if (umap[i] == id) idx.push_back(i);
      run_group(extract(A, idx, idx), idx);
    }
  }
  Index nc = 0;
  std::vector<Index> rank(n, -1);
  for (Index i = 0; i < n; ++i)
    if (is_c[i]) {
      rank[i] = nc++;
      out.C.push_back(i);
    } else {
      out.F.push_back(i);
    }
  if (nc == n) {
    out.stalled = true;
    return out;
  }
  std::vector<Triplet> e;
  e.reserve(local.size());
  for (size_t g = 0; g < groups.size(); ++g)
    for (size_t t = groups[g].second; t < group_end[g]; ++t)
      e.push_back({local[t].r, rank[group_c[g][local[t].c]], local[t].v});
  out.P = from_triplets(n, nc, e);
  if (!umap.empty()) {
    out.coarse_unknowns.resize(nc);
    for (Index k = 0; k < nc; ++k) out.coarse_unknowns[k] = umap[out.C[k]];
  }
  return out;
}

Vec vcycle(const AmgHierarchy& H, Index l, const Vec& r) {  // amg.cpp:232-242
  const AmgLevel& L = H.levels[l];
  if (l == H.num_levels() - 1) return H.coarse_solver.solve(r);
  Vec z = L.pre.apply(r);
  const Vec rc = spmv(L.R, sub(r, spmv(L.A, z)));
  const Vec ec = vcycle(H, l + 1, rc);
  spmv_add(L.P, ec, z);
  const Vec zp = L.post.apply(sub(r, spmv(L.A, z)));
  for (size_t i = 0; i < z.size(); ++i) z[i] += zp[i];
  return z;
}

}  // namespace

AmgHierarchy amg_setup(const Csr& A, const AmgConfig& cfg) {  // amg.cpp:246-291
  if (A.rows != A.cols) throw std::invalid_argument("amg_setup: matrix must be square");
  if (!(cfg.strength_theta > 0.0 && cfg.strength_theta < 1.0))
    throw std::invalid_argument("amg_setup: strength_theta must lie in (0,1)");
  if (cfg.coarse_size < 1) throw std::invalid_argument("amg_setup: coarse_size must be >= 1");
  if (!cfg.unknown_map.empty() && static_cast<Index>(cfg.unknown_map.size()) != A.rows)
    throw std::invalid_argument("amg_setup: unknown_map size mismatch");
  AmgHierarchy H;
  Csr Acur = A;
  std::vector<int> map = cfg.unknown_map;
  while (true) {
    const Index n = Acur.rows;
    H.info.level_sizes.push_back(n);
    AmgLevel L;
    L.A = Acur;
    L.unknown_map = map;
    const bool last = H.num_levels() + 1 >= cfg.max_levels;
    if (n <= cfg.coarse_size || last) {
      H.levels.push_back(std::move(L));
      break;
    }
    LevelInterp li = level_interp(Acur, cfg, map, &H.info.interp_fallback_rows);
    if (li.stalled) {
      H.info.truncated = true;
      H.levels.push_back(std::move(L));
      break;
    }
    L.P = li.P;
    L.R = transpose(li.P);
    L.C = li.C;
    L.F = li.F;
    L.pre = BoundSmoother::bind(cfg.pre_smoother, Acur);
    L.post = BoundSmoother::bind(cfg.post_smoother, Acur);
    Csr Anext = matmul(L.R, matmul(Acur, L.P));
    H.levels.push_back(std::move(L));
    Acur = std::move(Anext);
    map = std::move(li.coarse_unknowns);
  }
  H.coarse_solver = factor_dense(H.levels.back().A);
  return H;
}

Vec amg_vcycle(const AmgHierarchy& H, const Vec& r) {
  if (H.levels.empty()) throw std::logic_error("amg_vcycle: empty hierarchy");
  if (static_cast<Index>(r.size()) != H.fine_size())
    throw std::invalid_argument("amg_vcycle: residual size mismatch");
  return vcycle(H, 0, r);
}

// ============================================================================
// krylov — proj/src/krylov.cpp
// ============================================================================
namespace {

void givens(std::vector<Real>& H, Index ld, std::vector<Real>& cs, std::vector<Real>& sn,
            std::vector<Real>& g, Index k) {  // krylov.cpp:11-33
  auto h = [&](Index i, Index j) -> Real& { return H[static_cast<size_t>(j) * ld + i]; };
  for (Index i = 0; i < k; ++i) {
    const Real t = cs[i] * h(i, k) + sn[i] * h(i + 1, k);
    h(i + 1, k) = -sn[i] * h(i, k) + cs[i] * h(i + 1, k);
    h(i, k) = t;
  }
  const Real a = h(k, k), b = h(k + 1, k);
  const Real r = std::hypot(a, b);
  if (r == 0.0) {
    cs[k] = 1.0;
    sn[k] = 0.0;
  } else {
    cs[k] = a / r;
    sn[k] = b / r;
  }
  h(k, k) = r;
  h(k + 1, k) = 0.0;
  const Real t = cs[k] * g[k];
  g[k + 1] = -sn[k] * g[k];
  g[k] = t;
}

}  // namespace

SolveReport gmres_op(const LinOp& A, Index n, const Vec& b, Vec& x, const KrylovConfig& cfg,
                     const LinOp& M) {
  if (static_cast<Index>(b.size()) != n) throw std::invalid_argument("gmres: rhs size mismatch");
  if (static_cast<Index>(x.size()) != n) throw std::invalid_argument("gmres: initial guess size mismatch");
  if (cfg.restart < 1) throw std::invalid_argument("gmres: restart must be >= 1");
  for (Real v : b)
    if (!std::isfinite(v)) throw std::runtime_error("gmres: rhs contains non-finite entries");
  SolveReport rep;
  const Real bnorm = norm(b);
  if (bnorm == 0.0) {
    std::fill(x.begin(), x.end(), 0.0);
    rep.converged = true;
    return rep;
  }
  const Real target = std::max(cfg.rel_tol * bnorm, cfg.abs_tol);
  auto prec = [&](const Vec& v) -> Vec { return M ? M(v) : v; };
  const Index m = cfg.restart;
  const Index ld = m + 1;
  std::vector<Vec> V(m + 1);
  std::vector<Real> H(static_cast<size_t>(ld) * m, 0.0);
  auto h = [&](Index i, Index j) -> Real& { return H[static_cast<size_t>(j) * ld + i]; };
  std::vector<Real> cs(m, 0.0), sn(m, 0.0), g(m + 1, 0.0);
  const Real sqrt2 = std::sqrt(2.0);

  while (rep.iterations < cfg.max_iters) {
    Vec r = sub(b, A(x));
    const Real rnorm = norm(r);
    if (!std::isfinite(rnorm)) throw std::runtime_error("gmres: residual is non-finite");
    if (rnorm <= target) {
      rep.converged = true;
      rep.final_residual = rnorm / bnorm;
      rep.residual_history.push_back(rep.final_residual);
      return rep;
    }
    V[0].resize(n);
    for (Index i = 0; i < n; ++i) V[0][i] = r[i] / rnorm;
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = rnorm;
    Index k = 0;
    bool breakdown = false;
    for (; k < m && rep.iterations < cfg.max_iters; ++k) {
      Vec w = A(prec(V[k]));
      const Real w0 = norm(w);
      for (Index i = 0; i <= k; ++i) {
        const Real hh = dot(V[i], w);
        h(i, k) = hh;
        for (Index q = 0; q < n; ++q) w[q] -= hh * V[i][q];
      }
      if (norm(w) < w0 / sqrt2) {
        for (Index i = 0; i <= k; ++i) {
          const Real hh = dot(V[i], w);
          h(i, k) += hh;
          for (Index q = 0; q < n; ++q) w[q] -= hh * V[i][q];
        }
      }
      h(k + 1, k) = norm(w);
      if (!std::isfinite(h(k + 1, k))) throw std::runtime_error("gmres: Arnoldi vector is non-finite");
      const bool happy = h(k + 1, k) < 1e-300;
      if (!happy) {
        V[k + 1].resize(n);
        for (Index q = 0; q < n; ++q) V[k + 1][q] = w[q] / h(k + 1, k);
      }
      givens(H, ld, cs, sn, g, k);
      ++rep.iterations;
      const Real est = std::abs(g[k + 1]);
      rep.residual_history.push_back(est / bnorm);
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
    Index keff = k;
    while (keff > 0 && std::abs(h(keff - 1, keff - 1)) < 1e-300) --keff;
    if (keff > 0) {
      std::vector<Real> y(keff);
      for (Index i = keff - 1; i >= 0; --i) {
        Real s = g[i];
        for (Index j = i + 1; j < keff; ++j) s -= h(i, j) * y[j];
        y[i] = s / h(i, i);
      }
      Vec upd(n, 0.0);
      for (Index j = 0; j < keff; ++j)
        for (Index q = 0; q < n; ++q) upd[q] += V[j][q] * y[j];
      const Vec c = prec(upd);
      for (Index q = 0; q < n; ++q) x[q] += c[q];
    }
    const Vec rt = sub(b, A(x));
    const Real tn = norm(rt);
    if (!std::isfinite(tn)) throw std::runtime_error("gmres: residual is non-finite");
    rep.residual_history.push_back(tn / bnorm);
    if (tn <= target) {
      rep.converged = true;
      rep.final_residual = tn / bnorm;
      return rep;
    }
    if (breakdown) throw std::runtime_error("gmres: Arnoldi breakdown before reaching tolerance");
    rep.final_residual = tn / bnorm;
  }
  return rep;
}

SolveReport gmres(const Csr& A, const Vec& b, Vec& x, const KrylovConfig& cfg, const LinOp& M) {
  if (A.rows != A.cols) throw std::invalid_argument("gmres: matrix must be square");
  const LinOp op = [&A](const Vec& v) -> Vec { return spmv(A, v); };
  return gmres_op(op, A.rows, b, x, cfg, M);
}

// ============================================================================
// mgr — proj/src/mgr.cpp
// ============================================================================
DofPartition DofPartition::from_names(std::vector<std::string> order,
                                      const std::vector<std::string>& names) {
  DofPartition p;
  p.field_order = std::move(order);
  for (const auto& s : names) p.labels.push_back(p.field_id(s));
  return p;
}

Index DofPartition::field_id(const std::string& name) const {
  for (Index k = 0; k < static_cast<Index>(field_order.size()); ++k)
    if (field_order[k] == name) return k;
  throw std::invalid_argument("unknown field name: " + name);
}

namespace {

void split_ids(const std::vector<Index>& labels, const std::vector<char>& is_f, IndexList& F,
               IndexList& C) {  // mgr.cpp:27-35
  F.clear();
  C.clear();
  for (Index i = 0; i < static_cast<Index>(labels.size()); ++i) (is_f[labels[i]] ? F : C).push_back(i);
  if (F.empty()) throw std::invalid_argument("split: F set is empty");
  if (C.empty()) throw std::invalid_argument("split: C set is empty (all fields eliminated)");
}

std::vector<char> field_mask(const DofPartition& p, const std::vector<std::string>& f) {
  if (f.empty()) throw std::invalid_argument("split: f_fields must be nonempty");
  std::vector<char> m(p.field_order.size(), 0);
  for (const auto& s : f) m[p.field_id(s)] = 1;
  return m;
}

Csr ff_solve(const Csr& Aff, const Csr& B, const BlockLayout* layout) {  // mgr.cpp:46-65
  if (structurally_diagonal(Aff)) {
    const Vec dinv = diag_inverse(Aff);
    Csr X = B;
    for (Index i = 0; i < X.rows; ++i)
      for (Index k = X.ptr[i]; k < X.ptr[i + 1]; ++k) X.val[k] *= dinv[i];
    return X;
  }
  if (layout) return BlockDiagonalLU(Aff, *layout).solve_columns(B);
  if (Aff.rows <= 2000) {
    const DenseLU lu = factor_dense(Aff);
    return dense_to_sparse(lu.solve(to_dense(B)));
  }
  throw std::runtime_error(
      "ideal transfer operators require a structurally diagonal A_FF, a declared block "
      "layout, or |F| <= 2000 for a dense factorization");
}

void check_sets(Index n, const IndexList& F, const IndexList& C) {  // mgr.cpp:67-79
  std::vector<char> seen(n, 0);
  for (const IndexList* s : {&F, &C})
    for (Index i : *s) {
      if (i < 0 || i >= n || seen[i]) throw std::invalid_argument("F/C sets do not partition dofs");
      seen[i] = 1;
    }
  if (static_cast<Index>(F.size() + C.size()) != n)
    throw std::invalid_argument("F/C sets do not partition dofs");
}

template <typename T>
std::vector<T> gather(const std::vector<T>& v, const IndexList& idx) {
  std::vector<T> o;
  o.reserve(idx.size());
  for (Index i : idx) o.push_back(v[i]);
  return o;
}

}  // namespace

void split(const DofPartition& p, const std::vector<std::string>& f, IndexList& F, IndexList& C) {
  split_ids(p.labels, field_mask(p, f), F, C);
}

Csr build_interp(const Csr& A, const IndexList& F, const IndexList& C, InterpKind kind,
                 const BlockLayout* layout) {
  const Index n = A.rows;
  check_sets(n, F, C);
  const Index nf = static_cast<Index>(F.size()), nc = static_cast<Index>(C.size());
  const Csr Afc = extract(A, F, C);
  Csr W;
  if (kind == InterpKind::jacobi) {
    const Vec dinv = diag_inverse(extract(A, F, F));
    W = Afc;
    for (Index i = 0; i < nf; ++i)
      for (Index k = W.ptr[i]; k < W.ptr[i + 1]; ++k) W.val[k] *= dinv[i];
  } else {
    W = ff_solve(extract(A, F, F), Afc, layout);
  }
  std::vector<Triplet> e;
  for (Index i = 0; i < nf; ++i)
    for (Index k = W.ptr[i]; k < W.ptr[i + 1]; ++k) e.push_back({F[i], W.col[k], -W.val[k]});
  for (Index j = 0; j < nc; ++j) e.push_back({C[j], j, 1.0});
  return from_triplets(n, nc, e);
}

Csr build_restrict(const Csr& A, const IndexList& F, const IndexList& C, RestrictKind kind,
                   const BlockLayout* layout) {
  const Index n = A.rows;
  check_sets(n, F, C);
  const Index nc = static_cast<Index>(C.size());
  std::vector<Triplet> e;
  if (kind != RestrictKind::injection) {
    const Csr Acf = extract(A, C, F);
    Csr Z;
    if (kind == RestrictKind::jacobi) {
      const Vec dinv = diag_inverse(extract(A, F, F));
      Z = Acf;
      for (Index i = 0; i < nc; ++i)
        for (Index k = Z.ptr[i]; k < Z.ptr[i + 1]; ++k) Z.val[k] *= dinv[Z.col[k]];
    } else {
      Z = transpose(ff_solve(transpose(extract(A, F, F)), transpose(Acf), layout));
    }
    for (Index i = 0; i < nc; ++i)
      for (Index k = Z.ptr[i]; k < Z.ptr[i + 1]; ++k) e.push_back({i, F[Z.col[k]], -Z.val[k]});
  }
  for (Index j = 0; j < nc; ++j) e.push_back({j, C[j], 1.0});
  return from_triplets(nc, n, e);
}

Csr coarse_operator(const Csr& A, const Csr& R, const Csr& P) {
  if (R.cols != A.rows || A.cols != P.rows || R.rows != P.cols)
    throw std::invalid_argument("coarse_operator: dimension mismatch");
  return matmul(R, matmul(A, P));
}

Csr schur_jacobi_direct(const Csr& A, const IndexList& F, const IndexList& C) {
  check_sets(A.rows, F, C);
  const Csr Acc = extract(A, C, C), Afc = extract(A, F, C);
  Csr Acf = extract(A, C, F);
  const Vec dinv = diag_inverse(extract(A, F, F));
  for (Index i = 0; i < Acf.rows; ++i)
    for (Index k = Acf.ptr[i]; k < Acf.ptr[i + 1]; ++k) Acf.val[k] *= dinv[Acf.col[k]];
  const Csr M = matmul(Acf, Afc);
  std::vector<Triplet> t;
  for (Index i = 0; i < Acc.rows; ++i) {
    for (Index k = Acc.ptr[i]; k < Acc.ptr[i + 1]; ++k) t.push_back({i, Acc.col[k], Acc.val[k]});
    for (Index k = M.ptr[i]; k < M.ptr[i + 1]; ++k) t.push_back({i, M.col[k], -M.val[k]});
  }
  return from_triplets(Acc.rows, Acc.cols, t);
}

namespace {

Vec coarse_solve(const MgrHierarchy& H, const Vec& v) {  // mgr.cpp:177-194
  switch (H.coarse_spec.kind) {
    case CoarseSolverSpec::Kind::dense_lu:
      return H.coarse_lu.solve(v);
    case CoarseSolverSpec::Kind::amg_vcycle: {
      Vec z = amg_vcycle(*H.coarse_amg, v);
      for (Index c = 1; c < H.coarse_spec.amg_cycles; ++c) {
        const Vec d = amg_vcycle(*H.coarse_amg, sub(v, spmv(H.A_coarse, z)));
        for (size_t i = 0; i < z.size(); ++i) z[i] += d[i];
      }
      return z;
    }
    case CoarseSolverSpec::Kind::gmres_inner: {
      Vec x(v.size(), 0.0);
      gmres(H.A_coarse, v, x, H.coarse_spec.krylov);
      return x;
    }
  }
  throw std::logic_error("coarse_solve: unreachable");
}

Vec apply_level(const MgrHierarchy& H, Index l, const Vec& v) {  // mgr.cpp:196-219
  if (l == H.num_reduction_levels()) return coarse_solve(H, v);
  const MgrLevel& L = H.levels[l];
  Vec z;
  if (L.global_relax)
    z = L.global_relax->apply(v);
  else
    z.assign(v.size(), 0.0);
  {
    const Vec r = L.global_relax ? sub(v, spmv(L.A, z)) : v;
    Vec rF(L.F.size());
    for (size_t i = 0; i < L.F.size(); ++i) rF[i] = r[L.F[i]];
    const Vec zF = L.f_relax.apply(rF);
    for (size_t i = 0; i < L.F.size(); ++i) z[L.F[i]] += zF[i];
  }
  const Vec rc = spmv(L.R, sub(v, spmv(L.A, z)));
  const Vec e = apply_level(H, l + 1, rc);
  spmv_add(L.P, e, z);
  return z;
}

}  // namespace

MgrHierarchy mgr_setup(const Csr& A, const DofPartition& part, const MgrStrategy& strat,
                       const std::vector<int>* unknown_map) {
  if (A.rows != A.cols) throw std::invalid_argument("mgr_setup: matrix must be square");
  if (static_cast<Index>(part.labels.size()) != A.rows)
    throw std::invalid_argument("mgr_setup: partition size does not match the matrix");
  if (unknown_map && static_cast<Index>(unknown_map->size()) != A.rows)
    throw std::invalid_argument("mgr_setup: unknown_map size mismatch");
  {
    std::unordered_set<std::string> used;
    for (const auto& spec : strat.levels) {
      if (spec.f_fields.empty()) throw std::invalid_argument("mgr_setup: a level with no f_fields");
      for (const auto& f : spec.f_fields) {
        part.field_id(f);
        if (!used.insert(f).second) throw std::invalid_argument("mgr_setup: field eliminated twice: " + f);
      }
    }
  }
  MgrHierarchy H;
  H.coarse_spec = strat.coarse;
  Csr Acur = A;
  std::vector<Index> labels = part.labels;
  IndexList finest(A.rows);
  std::iota(finest.begin(), finest.end(), 0);
  std::vector<int> umap;
  if (unknown_map) umap = *unknown_map;
  for (const auto& spec : strat.levels) {
    MgrLevel L;
    L.A = Acur;
    L.finest_ids = finest;
    split_ids(labels, field_mask(part, spec.f_fields), L.F, L.C);
    BlockLayout layout;
    const BlockLayout* lp = nullptr;
    if (spec.ff_block_sizes) {
      layout = BlockLayout::from_sizes(*spec.ff_block_sizes);
      lp = &layout;
    }
    L.P = build_interp(Acur, L.F, L.C, spec.interp, lp);
    L.R = build_restrict(Acur, L.F, L.C, spec.restrict_kind, lp);
    const Csr Aff = extract(Acur, L.F, L.F);
    std::vector<int> uf;
    const std::vector<int>* ufp = nullptr;
    if (!umap.empty()) {
      uf = gather(umap, L.F);
      ufp = &uf;
    }
    L.f_relax = BoundSmoother::bind(spec.f_relax, Aff, ufp);
    if (spec.global_relax)
      L.global_relax = BoundSmoother::bind(*spec.global_relax, Acur, umap.empty() ? nullptr : &umap);
    Csr Anext = coarse_operator(Acur, L.R, L.P);
    labels = gather(labels, L.C);
    finest = gather(finest, L.C);
    if (!umap.empty()) umap = gather(umap, L.C);
    H.levels.push_back(std::move(L));
    Acur = std::move(Anext);
  }
  H.A_coarse = Acur;
  H.coarse_finest_ids = finest;
  H.coarse_unknown_map = umap;
  switch (strat.coarse.kind) {
    case CoarseSolverSpec::Kind::dense_lu:
      H.coarse_lu = factor_dense(H.A_coarse);
      break;
    case CoarseSolverSpec::Kind::amg_vcycle: {
      AmgConfig cfg = strat.coarse.amg;
      if (strat.coarse.use_unknown_map) {
        if (umap.empty())
          throw std::invalid_argument("mgr_setup: coarse solver requests an unknown map, none given");
        cfg.unknown_map = umap;
      }
      H.coarse_amg = std::make_shared<AmgHierarchy>(amg_setup(H.A_coarse, cfg));
      break;
    }
    case CoarseSolverSpec::Kind::gmres_inner:
      break;
  }
  return H;
}

Vec mgr_apply(const MgrHierarchy& H, const Vec& v) {
  if (static_cast<Index>(v.size()) != H.fine_size()) throw std::invalid_argument("mgr_apply: size mismatch");
  return apply_level(H, 0, v);
}

LinOp mgr_preconditioner(const MgrHierarchy& H) {
  const MgrHierarchy* h = &H;
  return [h](const Vec& v) -> Vec { return mgr_apply(*h, v); };
}

}  // namespace refcpu
