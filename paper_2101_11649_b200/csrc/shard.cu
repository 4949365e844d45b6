// Row-slab sharded MGR-GMRES. See shard.cuh.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "shard.cuh"

namespace mgrx {
namespace {

__global__ void k_pack(int n, const int* __restrict__ idx, const double* __restrict__ x, double* __restrict__ y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = x[idx[i]];
}
__global__ void k_scatter_add_s(int n, const int* __restrict__ idx, const double* __restrict__ a,
                                double* __restrict__ y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[idx[i]] = __dadd_rn(y[idx[i]], a[i]);
}
// Sum of the per-rank partials (pairs) in rank order; every rank folds the
// same gathered values in the same order, so all ranks hold the same bits.
__global__ void k_fold2(int size, const double* __restrict__ g, double* dh, double* hacc, int acc, double* dn) {
  double v0 = g[0], v1 = g[1];
  for (int q = 1; q < size; ++q) {
    v0 = __dadd_rn(v0, g[2 * q]);
    v1 = __dadd_rn(v1, g[2 * q + 1]);
  }
  if (dh) *dh = v0;
  if (hacc) *hacc = acc ? __dadd_rn(*hacc, v0) : v0;
  if (dn) *dn = v1;
}

void fold2(int size, const double* g, double* dh, double* hacc, bool acc, double* dn, cudaStream_t s) {
  k_fold2<<<1, 1, 0, s>>>(size, g, dh, hacc, acc ? 1 : 0, dn);
  MGRX_LAUNCH_CK();
  count_launch();
}

void pack(int n, const int* idx, const double* x, double* y, cudaStream_t s) {
  if (n <= 0) return;
  k_pack<<<blocks_for(n, 256), 256, 0, s>>>(n, idx, x, y);
  MGRX_LAUNCH_CK();
  count_launch();
}

void d2d(double* dst, const double* src, int n, cudaStream_t s) {
  if (n > 0) MGRX_CK(cudaMemcpyAsync(dst, src, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
}

template <class T>
std::vector<T> dl(const DVec<T>& v, size_t n, cudaStream_t s) {
  std::vector<T> h(n);
  if (n) {
    MGRX_CK(cudaMemcpyAsync(h.data(), v.get(), n * sizeof(T), cudaMemcpyDeviceToHost, s));
    MGRX_CK(cudaStreamSynchronize(s));
  }
  return h;
}

// st[q] = number of entries of the ascending list `sub` below p.st[q]
Part sub_part(const Part& p, const std::vector<int>& sub) {
  Part o;
  o.st.resize(p.st.size());
  for (size_t q = 0; q < p.st.size(); ++q)
    o.st[q] = static_cast<int>(std::lower_bound(sub.begin(), sub.end(), p.st[q]) - sub.begin());
  o.st.back() = static_cast<int>(sub.size());
  return o;
}

Space make_space(const Part& p, int rank) {
  Space s;
  s.part = p;
  s.own = p.n(rank);
  s.cap = s.own;
  return s;
}

// Slab of global operator G: rows of `rows` owned by `rank`, columns of the
// space `cols` renumbered [owned | halo]. The send lists are derived from the
// other ranks' rows of the same (replicated) operator.
void build_op(SOp& op, const DCsr& G, const Part& rows, Space& cols, int rank, cudaStream_t s) {
  const int size = static_cast<int>(rows.st.size()) - 1;
  if (G.rows != rows.total() || G.cols != cols.part.total())
    throw RuntimeError("sharded solve: operator does not match its index spaces");
  const std::vector<int> ptr = dl(G.ptr, G.rows + 1, s);
  const std::vector<int> col = dl(G.col, G.nnz, s);
  const std::vector<double> val = dl(G.val, G.nnz, s);
  const int r0 = rows.lo(rank), r1 = rows.hi(rank);
  const int c0 = cols.part.lo(rank), c1 = cols.part.hi(rank);
  op.own = c1 - c0;
  // halo of this rank: sorted unique non-owned columns of its rows
  std::vector<int> halo;
  for (int k = ptr[r0]; k < ptr[r1]; ++k)
    if (col[k] < c0 || col[k] >= c1) halo.push_back(col[k]);
  std::sort(halo.begin(), halo.end());
  halo.erase(std::unique(halo.begin(), halo.end()), halo.end());
  op.nhalo = static_cast<int>(halo.size());
  cols.need(op.nhalo);
  // local CSR (entries keep their order: the per-row sum is unchanged)
  const int m = r1 - r0;
  std::vector<int> lp(m + 1), lc(ptr[r1] - ptr[r0]);
  std::vector<double> lv(val.begin() + ptr[r0], val.begin() + ptr[r1]);
  for (int i = 0; i <= m; ++i) lp[i] = ptr[r0 + i] - ptr[r0];
  for (int k = ptr[r0]; k < ptr[r1]; ++k) {
    const int j = col[k];
    lc[k - ptr[r0]] = (j >= c0 && j < c1)
                          ? j - c0
                          : op.own + static_cast<int>(std::lower_bound(halo.begin(), halo.end(), j) - halo.begin());
  }
  op.M = DCsr();
  op.M.rows = m;
  op.M.cols = op.own + op.nhalo;
  op.M.nnz = static_cast<int>(lc.size());
  op.M.ptr.alloc(m + 1, s);
  op.M.ptr.upload(lp.data(), m + 1);
  op.M.col.alloc(lc.size() > 0 ? lc.size() : 1, s);
  op.M.col.upload(lc.data(), lc.size());
  op.M.val.alloc(lv.size() > 0 ? lv.size() : 1, s);
  op.M.val.upload(lv.data(), lv.size());
  // recv segments: halo entries grouped by owner (owners are monotone in j)
  op.recv.clear();
  for (int a = 0; a < op.nhalo;) {
    const int q = cols.part.owner(halo[a]);
    int b = a;
    while (b < op.nhalo && halo[b] < cols.part.hi(q)) ++b;
    op.recv.push_back({q, a, b - a});
    a = b;
  }
  // send segments: for every other rank q, the owned columns its rows read
  op.send.clear();
  std::vector<int> sidx;
  for (int q = 0; q < size; ++q) {
    if (q == rank) continue;
    std::vector<int> need;
    for (int k = ptr[rows.lo(q)]; k < ptr[rows.hi(q)]; ++k)
      if (col[k] >= c0 && col[k] < c1) need.push_back(col[k] - c0);
    if (need.empty()) continue;
    std::sort(need.begin(), need.end());
    need.erase(std::unique(need.begin(), need.end()), need.end());
    op.send.push_back({q, static_cast<int>(sidx.size()), static_cast<int>(need.size())});
    sidx.insert(sidx.end(), need.begin(), need.end());
  }
  op.sidx.alloc(sidx.size() > 0 ? sidx.size() : 1, s);
  op.sidx.upload(sidx.data(), sidx.size());
  op.sbuf.alloc(sidx.size() > 0 ? sidx.size() : 1, s);
  op.built = true;
  spmv_prepare(op.M, s);
}

// Fill the halo region x[own, own + nhalo) of an extended vector.
void halo(SOp& op, double* x, ShardCtx& c) {
  if (c.size == 1) return;
  int tot = 0;
  for (const Seg& g : op.send) tot += g.count;
  pack(tot, op.sidx.get(), x, op.sbuf.get(), c.s);
  std::vector<Xfer> sends, recvs;
  for (const Seg& g : op.send) sends.push_back({g.peer, op.sbuf.get() + g.off, g.count});
  for (const Seg& g : op.recv) recvs.push_back({g.peer, x + op.own + g.off, g.count});
  c.comm->exchange(sends, recvs, c.s);
}

DVec<int> upload_ints(const std::vector<int>& v, cudaStream_t s) {
  DVec<int> d(v.size() > 0 ? v.size() : 1, s);
  d.upload(v.data(), v.size());
  return d;
}

void alloc_cap(DVec<double>& v, const Space& sp, cudaStream_t s) { v.alloc(sp.cap > 0 ? sp.cap : 1, s); }

}  // namespace

int Part::owner(int g) const {
  return static_cast<int>(std::upper_bound(st.begin(), st.end(), g) - st.begin()) - 1;
}

// ---------------------------------------------------------------------------
// replicated dense solve
// ---------------------------------------------------------------------------
void Repl::build(const DenseLU* f, const Part& p, cudaStream_t s) {
  lu = f;
  part = p;
  const int size = static_cast<int>(p.st.size()) - 1;
  maxc = 1;
  for (int q = 0; q < size; ++q) maxc = std::max(maxc, p.n(q));
  std::vector<int> m(p.total());
  for (int q = 0; q < size; ++q)
    for (int g = p.lo(q); g < p.hi(q); ++g) m[g] = q * maxc + (g - p.lo(q));
  map = upload_ints(m, s);
  pad.alloc(maxc, s);
  pad.zero();
  all.alloc(static_cast<size_t>(size) * maxc, s);
  full.alloc(p.total() > 0 ? p.total() : 1, s);
  sol.alloc(p.total() > 0 ? p.total() : 1, s);
}

void Repl::solve(const double* r, double* z, ShardCtx& c) {
  const int own = part.n(c.rank);
  d2d(pad.get(), r, own, c.s);
  c.comm->allgather(pad.get(), all.get(), maxc, c.s);
  pack(part.total(), map.get(), all.get(), full.get(), c.s);
  dense_solve(*lu, full.get(), sol.get(), c.s);
  d2d(z, sol.get() + part.lo(c.rank), own, c.s);
}

// ---------------------------------------------------------------------------
// smoothers
// ---------------------------------------------------------------------------
void SRelax::build(const BoundRelax& g, const DCsr& Ag, Space& space, ShardCtx& c) {
  kind = g.spec.kind;
  sweeps = g.spec.sweeps;
  weight = g.spec.weight;
  sp = &space;
  n = space.own;
  const int lo = space.part.lo(c.rank);
  switch (kind) {
    case Smoother::jacobi:
    case Smoother::l1_jacobi:
      dinv.alloc(n > 0 ? n : 1, c.s);
      d2d(dinv.get(), g.dinv.get() + lo, n, c.s);
      if (sweeps > 1) build_op(A, Ag, space.part, space, c.rank, c.s);
      break;
    case Smoother::amg_vcycle:
      amg = std::make_unique<SAmg>();
      amg->build(*g.amg, space, c);
      if (sweeps > 1) build_op(A, Ag, space.part, space, c.rank, c.s);
      break;
    case Smoother::dense_lu:
      dense.build(&g.lu, space.part, c.s);
      break;
    case Smoother::hybrid_l1_gs_forward:
    case Smoother::hybrid_l1_gs_backward:
      throw RuntimeError(
          "sharded solve: hybrid Gauss-Seidel is a sequential sweep over the whole matrix; use a "
          "Jacobi-family or AMG smoother");
    default:
      throw RuntimeError("sharded solve: smoother kind not supported across slabs");
  }
}

void SRelax::alloc(cudaStream_t s) {
  alloc_cap(b0, *sp, s);
  alloc_cap(b1, *sp, s);
  alloc_cap(b2, *sp, s);
  if (amg) alloc_cap(b3, *sp, s);
  if (amg) amg->alloc(s);
}

void SRelax::apply(const double* r, const int* rrow, double* z, double* zacc, ShardCtx& c) {
  if (kind == Smoother::jacobi || kind == Smoother::l1_jacobi) {
    // sweep 0: z = w*(dinv*r); later: z += w*(dinv*(r - A z)) (relax.cpp:168-174)
    if (sweeps == 1) {
      double* out = zacc ? b0.get() : z;
      jacobi0(n, weight, dinv.get(), r, rrow, out, c.s);
      if (zacc) vec_add(n, out, zacc, c.s);
      return;
    }
    jacobi0(n, weight, dinv.get(), r, rrow, b0.get(), c.s);
    double* cur = b0.get();
    double* bufs[2] = {b1.get(), b2.get()};
    for (int sw = 1; sw < sweeps; ++sw) {
      const bool last = sw == sweeps - 1;
      double* nxt = last ? (zacc ? nullptr : z) : bufs[sw % 2];
      halo(A, cur, c);
      spmv_jacobi_ex(A.M, cur, r, rrow, dinv.get(), weight, nxt, last ? zacc : nullptr, c.s);
      cur = nxt;
    }
    return;
  }
  const double* rin = r;
  if (rrow) {
    if (n > 0) gather(n, rrow, r, b2.get(), c.s);
    rin = b2.get();
  }
  double* out = zacc ? b0.get() : z;
  if (kind == Smoother::dense_lu) {
    dense.solve(rin, out, c);
  } else {
    // z = V(r); z += V(r - A z) (relax.cpp:186-190)
    amg->vcycle(rin, out, c);
    for (int sw = 1; sw < sweeps; ++sw) {
      halo(A, out, c);
      spmv_residual(A.M, out, rin, nullptr, b1.get(), c.s);
      amg->vcycle(b1.get(), b3.get(), c);
      vec_add(n, b3.get(), out, c.s);
    }
  }
  if (zacc) vec_add(n, out, zacc, c.s);
}

// ---------------------------------------------------------------------------
// AMG
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// replicated coarse V-cycle
// ---------------------------------------------------------------------------
void RepAmg::build(const AmgHier& h, int l, const Part& p, cudaStream_t s) {
  g = &h;
  from = l;
  part = p;
  const int size = static_cast<int>(p.st.size()) - 1;
  maxc = 1;
  for (int q = 0; q < size; ++q) maxc = std::max(maxc, p.n(q));
  std::vector<int> m(p.total());
  for (int q = 0; q < size; ++q)
    for (int gr = p.lo(q); gr < p.hi(q); ++gr) m[gr] = q * maxc + (gr - p.lo(q));
  map = upload_ints(m, s);
  pad.alloc(maxc, s);
  pad.zero();
  all.alloc(static_cast<size_t>(size) * maxc, s);
  const int n0 = std::max(1, p.total());
  rfull.alloc(n0, s);
  zfull.alloc(n0, s);
  const int nl = static_cast<int>(h.levels.size());
  for (int k = l; k < nl; ++k) {
    lv.emplace_back();
    const int n = std::max(1, h.levels[k].A.rows);
    for (DVec<double>* v : {&lv.back().r, &lv.back().z, &lv.back().t, &lv.back().w1, &lv.back().w2}) v->alloc(n, s);
  }
}

// BoundRelax::apply / apply_add (Jacobi kinds, folded sweep 0: n <= 64K)
void RepAmg::smooth(const BoundRelax& b, const double* r, double* z, double* zacc, Lv& w, cudaStream_t s) {
  const int n = b.n;
  if (b.spec.sweeps <= 1) {
    double* out = zacc ? w.w1.get() : z;
    jacobi0(n, b.spec.weight, b.dinv.get(), r, nullptr, out, s);
    if (zacc) vec_add(n, out, zacc, s);
    return;
  }
  const double* cur = nullptr;
  double* bufs[2] = {w.w1.get(), w.w2.get()};
  for (int sw = 1; sw < b.spec.sweeps; ++sw) {
    const bool last = sw == b.spec.sweeps - 1;
    double* nxt = last ? (zacc ? nullptr : z) : bufs[sw % 2];
    spmv_jacobi_ex(*b.A, cur, r, nullptr, b.dinv.get(), b.spec.weight, nxt, last ? zacc : nullptr, s);
    cur = nxt;
  }
}

void RepAmg::level(int l, const double* r, double* z, cudaStream_t s) {
  const int nl = static_cast<int>(g->levels.size());
  if (l == g->tail) {
    launch_amg_tail(g->tail_desc, g->tail_blob.get(), r, z, s);
    return;
  }
  if (l == nl - 1) {
    dense_solve(g->coarse, r, z, s);
    return;
  }
  const AmgLevelD& G = g->levels[l];
  Lv& W = lv[l - from];
  Lv& N = lv[l + 1 - from];
  smooth(G.pre, r, z, nullptr, W, s);
  spmv_residual(G.A, z, r, nullptr, W.t.get(), s);
  spmv(G.R, W.t.get(), N.r.get(), s);
  level(l + 1, N.r.get(), N.z.get(), s);
  spmv_add(G.P, N.z.get(), z, s);
  spmv_residual(G.A, z, r, nullptr, W.t.get(), s);
  smooth(G.post, W.t.get(), nullptr, z, W, s);
}

void RepAmg::vcycle(const double* r, double* z, ShardCtx& c) {
  const int own = part.n(c.rank);
  d2d(pad.get(), r, own, c.s);
  c.comm->allgather(pad.get(), all.get(), maxc, c.s);
  pack(part.total(), map.get(), all.get(), rfull.get(), c.s);
  level(from, rfull.get(), zfull.get(), c.s);
  d2d(z, zfull.get() + part.lo(c.rank), own, c.s);
}

int repl_rows() {
  static const int m = [] {
    const char* v = std::getenv("MGRX_SHARD_REPL_ROWS");
    return v ? std::atoi(v) : 65536;
  }();
  return m;
}

void SAmg::build(const AmgHier& g, Space& fine, ShardCtx& c) {
  const int nl = static_cast<int>(g.levels.size());
  std::vector<Space*> sp(nl);
  sp[0] = &fine;
  for (int l = 1; l < nl; ++l) {
    const AmgLevelD& G = g.levels[l - 1];
    const std::vector<int> C = dl(G.C, G.P.cols, c.s);
    spaces.push_back(make_space(sub_part(sp[l - 1]->part, C), c.rank));
    sp[l] = &spaces.back();
  }
  // first level that is replicated: small, Jacobi-type smoothing from there
  // on (the single-GPU smoother path without a gather), more than one rank
  int from = -1;
  if (c.size > 1 && repl_rows() > 0) {
    for (int l = 1; l < nl && from < 0; ++l) {
      if (g.levels[l].A.rows > repl_rows()) continue;
      bool ok = true;
      for (int k = l; k < nl - 1 && ok; ++k) {
        const BoundRelax* bs[2] = {&g.levels[k].pre, &g.levels[k].post};
        for (const BoundRelax* b : bs)
          ok = ok && (b->spec.kind == Smoother::jacobi || b->spec.kind == Smoother::l1_jacobi) &&
               (b->spec.sweeps <= 1 || b->n <= fold_sweep0_max_rows());
      }
      if (ok) from = l;
    }
  }
  for (int l = 0; l < nl; ++l) {
    L.emplace_back();
    SAmgLevel& S = L.back();
    S.sp = sp[l];
    if (l == from) {
      rep.build(g, l, sp[l]->part, c.s);
      break;
    }
    if (l == nl - 1) {
      coarse.build(&g.coarse, sp[l]->part, c.s);
      break;
    }
    const AmgLevelD& G = g.levels[l];
    build_op(S.A, G.A, sp[l]->part, *sp[l], c.rank, c.s);
    build_op(S.R, G.R, sp[l + 1]->part, *sp[l], c.rank, c.s);
    build_op(S.P, G.P, sp[l]->part, *sp[l + 1], c.rank, c.s);
    S.pre.build(G.pre, G.A, *sp[l], c);
    S.post.build(G.post, G.A, *sp[l], c);
  }
}

void SAmg::alloc(cudaStream_t s) {
  for (size_t l = 0; l < L.size(); ++l) {
    SAmgLevel& S = L[l];
    alloc_cap(S.r, *S.sp, s);
    alloc_cap(S.z, *S.sp, s);
    alloc_cap(S.t, *S.sp, s);
    if (l + 1 < L.size()) {
      S.pre.alloc(s);
      S.post.alloc(s);
    }
  }
}

// V(1,1) (proj/src/amg.cpp:232-242), with halos before each product.
void SAmg::level(int l, const double* r, double* z, ShardCtx& c) {
  SAmgLevel& S = L[l];
  if (l == rep.from) {
    rep.vcycle(r, z, c);
    return;
  }
  if (l == static_cast<int>(L.size()) - 1) {
    coarse.solve(r, z, c);
    return;
  }
  SAmgLevel& N = L[l + 1];
  S.pre.apply(r, nullptr, z, nullptr, c);  // z = pre(r)
  halo(S.A, z, c);
  spmv_residual(S.A.M, z, r, nullptr, S.t.get(), c.s);  // t = r - A z
  halo(S.R, S.t.get(), c);
  spmv(S.R.M, S.t.get(), N.r.get(), c.s);  // rc = R t
  level(l + 1, N.r.get(), N.z.get(), c);
  halo(S.P, N.z.get(), c);
  spmv_add(S.P.M, N.z.get(), z, c.s);  // z += P ec
  halo(S.A, z, c);
  spmv_residual(S.A.M, z, r, nullptr, S.t.get(), c.s);  // t = r - A z
  S.post.apply(S.t.get(), nullptr, nullptr, z, c);      // z += post(t)
}

// ---------------------------------------------------------------------------
// MGR
// ---------------------------------------------------------------------------
void Shard::build(MgrHier& h, const DCsr& A, const std::vector<int>& fine_starts, std::unique_ptr<Comm> cm,
                  cudaStream_t stream) {
  comm = std::move(cm);
  c.comm = comm.get();
  c.rank = comm->rank;
  c.size = comm->size;
  c.s = stream;
  H = &h;
  Ag = &A;
  Part p0;
  p0.st = fine_starts;
  if (static_cast<int>(p0.st.size()) != c.size + 1 || p0.st.front() != 0 || p0.st.back() != A.rows)
    throw InvalidArgument("sharded solve: row starts must be size+1 offsets from 0 to n");
  for (int q = 0; q < c.size; ++q)
    if (p0.st[q + 1] <= p0.st[q]) throw InvalidArgument("sharded solve: every rank needs at least one row");
  row_begin = p0.lo(c.rank);
  row_end = p0.hi(c.rank);
  spaces.push_back(make_space(p0, c.rank));
  Space* cur = &spaces.back();
  for (auto& G : h.levels) {
    levels.emplace_back();
    SMgrLevel& S = levels.back();
    S.sl = cur;
    const int nf = static_cast<int>(G.F.size()), nc = static_cast<int>(G.C.size());
    const std::vector<int> F = dl(G.F, nf, c.s), C = dl(G.C, nc, c.s);
    spaces.push_back(make_space(sub_part(cur->part, F), c.rank));
    S.sf = &spaces.back();
    spaces.push_back(make_space(sub_part(cur->part, C), c.rank));
    S.sc = &spaces.back();
    const int lo = cur->part.lo(c.rank);
    S.nl = cur->own;
    S.nf = S.sf->own;
    S.nc = S.sc->own;
    std::vector<int> fl(S.nf), cl(S.nc);
    for (int i = 0; i < S.nf; ++i) fl[i] = F[S.sf->part.lo(c.rank) + i] - lo;
    for (int i = 0; i < S.nc; ++i) cl[i] = C[S.sc->part.lo(c.rank) + i] - lo;
    std::vector<int> fp(S.nl, -1);
    for (int i = 0; i < S.nf; ++i) fp[fl[i]] = i;
    S.Floc = upload_ints(fl, c.s);
    S.Cloc = upload_ints(cl, c.s);
    S.fpos = upload_ints(fp, c.s);
    S.injection = G.injection;
    S.general = !G.injection || G.g_relax.has_value();
    build_op(S.P, G.P, cur->part, *S.sc, c.rank, c.s);
    if (S.general) {
      build_op(S.A, G.A, cur->part, *cur, c.rank, c.s);
      build_op(S.R, G.R, S.sc->part, *cur, c.rank, c.s);
      if (G.g_relax) {
        S.g_relax = std::make_unique<SRelax>();
        S.g_relax->build(*G.g_relax, G.A, *cur, c);
      }
    } else {
      build_op(S.Acf, G.Acf, S.sc->part, *S.sf, c.rank, c.s);
    }
    S.f_relax.build(G.f_relax, G.Aff, *S.sf, c);
    cur = S.sc;
  }
  // coarse solver on the last C space
  if (h.coarse_spec.kind == Coarse::dense_lu) {
    coarse_lu.build(&h.coarse_lu, cur->part, c.s);
  } else {
    coarse_amg = std::make_unique<SAmg>();
    coarse_amg->build(*h.coarse_amg, *cur, c);
    coarse_cycles = h.coarse_spec.cycles;
    if (coarse_cycles > 1) build_op(Acoarse, h.A_coarse, cur->part, *cur, c.rank, c.s);
  }
  build_op(Afine, A, spaces.front().part, spaces.front(), c.rank, c.s);
  // buffers last: every space's halo capacity is known now
  for (auto& S : levels) {
    alloc_cap(S.zF, *S.sf, c.s);
    alloc_cap(S.vF, *S.sf, c.s);
    alloc_cap(S.rc, *S.sc, c.s);
    alloc_cap(S.e, *S.sc, c.s);
    alloc_cap(S.t, *S.sl, c.s);
    S.f_relax.alloc(c.s);
    if (S.g_relax) S.g_relax->alloc(c.s);
  }
  if (coarse_amg) coarse_amg->alloc(c.s);
  alloc_cap(ct, *cur, c.s);
  alloc_cap(cd, *cur, c.s);
  alloc_cap(xext, spaces.front(), c.s);
  alloc_cap(zext, spaces.front(), c.s);
  loc.alloc(2, c.s);
  loc.zero();
  gbuf.alloc(2 * c.size, c.s);
  MGRX_CK(cudaStreamSynchronize(c.s));
  setup_fused();
}

namespace {
// deterministic self-check data from the global row index
__global__ void k_seed(int n, int row0, int salt, double* v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const unsigned h = (static_cast<unsigned>(row0 + i) * 2654435761u) ^ (static_cast<unsigned>(salt) * 40503u);
    v[i] = static_cast<double>(h % 2000003u) / 2000003.0 - 0.5;
  }
}
}  // namespace

ArnoldiPeers Shard::peers_arg() {
  ArnoldiPeers pe;
  pe.nranks = c.size;
  pe.rank = c.rank;
  pe.mbox = mbox;
  pe.peers = peer_dev.get();
  epoch += 1ull << 16;
  pe.epoch = epoch;
  return pe;
}

void Shard::setup_fused() {
  fused = false;
  const char* fe = std::getenv("MGRX_SHARD_FUSED");
  if (fe && std::atoi(fe) == 0) return;
  // one rank: the exchange is the identity (k_fold2 of one partial is the
  // partial), so the single-GPU fused kernel is the same computation
  if (c.size == 1) {
    fused = arnoldi_sharded_ok(spaces.front().own);
    return;
  }
  // multi-rank in-kernel mailbox exchange: opt-in (MGRX_SHARD_FUSED=1) until
  // a multi-GPU run has validated it; the default sharded solve is the
  // low-synchronisation GMRES with two all-gathers per step
  if (!(fe && std::atoi(fe) == 1)) return;
  // ranks of the local comm share one device: the in-kernel exchange needs
  // every rank's persistent kernel resident at once, i.e. one GPU per rank
  if (c.size < 2 || c.size > kMboxRanks || std::string(comm->kind()) != "nccl") return;
  const int n = spaces.front().own;
  cudaStream_t s = c.s;
  auto agree = [&](bool mine) {  // min over ranks
    const double flag[2] = {mine ? 1.0 : 0.0, 0.0};
    loc.upload(flag, 2);
    c.comm->allgather(loc.get(), gbuf.get(), 2, s);
    const std::vector<double> g = gbuf.download(2 * c.size);
    bool all = true;
    for (int q = 0; q < c.size; ++q) all = all && g[2 * q] == 1.0;
    return all;
  };
  if (!agree(arnoldi_sharded_ok(n))) return;
  MGRX_CK(cudaMalloc(&mbox, sizeof(double) * kMboxDoubles));
  MGRX_CK(cudaMemset(mbox, 0, sizeof(double) * kMboxDoubles));
  if (!c.comm->map_peers(mbox, peer_mbox)) {
    cudaFree(mbox);
    mbox = nullptr;
    return;
  }
  std::vector<double*> pd(c.size);
  for (int q = 0; q < c.size; ++q) pd[q] = static_cast<double*>(peer_mbox[q]);
  peer_dev.alloc(c.size, s);
  peer_dev.upload(pd.data(), c.size);
  // self-check: one step (k = 1, both passes) through both paths
  const int m = 30, k = 1;
  ws.ensure(n, m, s);
  double* V = ws.V.get();
  for (int j = 0; j <= k; ++j) k_seed<<<blocks_for(n, 256), 256, 0, s>>>(n, row_begin, j + 1, V + static_cast<size_t>(j) * n);
  k_seed<<<blocks_for(n, 256), 256, 0, s>>>(n, row_begin, 7, ws.w.get());
  MGRX_LAUNCH_CK();
  DVec<double> w0(n, s);
  d2d(w0.get(), ws.w.get(), n, s);
  double* S = ws.scal.get();
  const int ns = 3 + 2 * (m + 1) + 1;
  arnoldi_sharded(n, k, 4, peers_arg(), ws, s);
  const std::vector<double> fusedS = ws.scal.download(ns);
  d2d(ws.w.get(), w0.get(), n, s);
  double* L = loc.get();
  auto reduce = [&](double* dh, double* hacc, bool acc, double* dn) {
    c.comm->allgather(L, gbuf.get(), 2, s);
    fold2(c.size, gbuf.get(), dh, hacc, acc, dn, s);
  };
  double* s_hp = S + 2;
  double* s_hc = S + 3 + (m + 1);
  for (int pass = 0; pass < 2; ++pass) {
    const bool second = pass == 1;
    for (int i = 0; i <= k; ++i) {
      mgs_step(n, ws.w.get(), i ? V + static_cast<size_t>(i - 1) * n : nullptr, i ? s_hp + (i - 1) : nullptr,
               V + static_cast<size_t>(i) * n, i == 0 && !second, ws, L, nullptr, false,
               (i == 0 && !second) ? L + 1 : nullptr, s);
      reduce(s_hp + i, s_hc + i, second, (i == 0 && !second) ? S : nullptr);
    }
    mgs_step(n, ws.w.get(), V + static_cast<size_t>(k) * n, s_hp + k, nullptr, true, ws, nullptr, nullptr, false,
             L + 1, s);
    reduce(nullptr, nullptr, false, S + 1);
  }
  const std::vector<double> ncclS = ws.scal.download(ns);
  bool same = fusedS[m + 3] == 0.0;  // no peer timeout
  for (int idx : {0, 1}) same = same && std::memcmp(&fusedS[idx], &ncclS[idx], sizeof(double)) == 0;
  for (int i = 0; i <= k; ++i)
    same = same && std::memcmp(&fusedS[3 + (m + 1) + i], &ncclS[3 + (m + 1) + i], sizeof(double)) == 0;
  fused = agree(same);
  if (const char* v = std::getenv("MGRX_VERBOSE"); v && v[0] == '1')
    std::fprintf(stderr, "[mgrx] shard %d/%d: fused sharded Arnoldi %s\n", c.rank, c.size,
                 fused ? "on (self-check bitwise equal)" : "off (self-check failed)");
  if (!fused) {
    c.comm->unmap_peers(peer_mbox);
    cudaFree(mbox);
    mbox = nullptr;
  }
}

Shard::~Shard() {
  if (mbox) {
    if (c.s) cudaStreamSynchronize(c.s);
    if (comm) comm->unmap_peers(peer_mbox);
    cudaFree(mbox);
  }
  if (graph) cudaGraphExecDestroy(graph);
  // buffers are freed on c.s by their destructors; the stream is destroyed
  // after them by the owning API object (mgrx_shard_destroy)
  if (c.s) cudaStreamSynchronize(c.s);
}

void Shard::coarse_solve(const double* v, double* z) {
  if (!coarse_amg) {
    coarse_lu.solve(v, z, c);
    return;
  }
  const int n = spaces.back().own;
  // z = V(v); z += V(v - A_c z) (mgr.cpp:181-186)
  coarse_amg->vcycle(v, z, c);
  for (int k = 1; k < coarse_cycles; ++k) {
    halo(Acoarse, z, c);
    spmv_residual(Acoarse.M, z, v, nullptr, ct.get(), c.s);
    coarse_amg->vcycle(ct.get(), cd.get(), c);
    vec_add(n, cd.get(), z, c.s);
  }
}

// Algorithm 1 (proj/src/mgr.cpp:196-219) on the owned rows; same fast path
// and operation order as MgrHier::apply_level.
void Shard::apply_level(int l, const double* v, double* z) {
  if (l == static_cast<int>(levels.size())) {
    coarse_solve(v, z);
    return;
  }
  SMgrLevel& S = levels[l];
  if (!S.general) {
    S.f_relax.apply(v, S.Floc.get(), S.zF.get(), nullptr, c);  // zF = f_relax(v_F)
    halo(S.Acf, S.zF.get(), c);
    spmv_residual(S.Acf.M, S.zF.get(), v, S.Cloc.get(), S.rc.get(), c.s);  // rc = v_C - A_CF zF
    apply_level(l + 1, S.rc.get(), S.e.get());
    halo(S.P, S.e.get(), c);
    spmv_prolong(S.P.M, S.e.get(), S.fpos.get(), S.zF.get(), z, c.s);  // z = [zF; 0] + P e
    return;
  }
  const double* r = v;
  if (S.g_relax) {
    S.g_relax->apply(v, nullptr, z, nullptr, c);
    halo(S.A, z, c);
    spmv_residual(S.A.M, z, v, nullptr, S.t.get(), c.s);
    r = S.t.get();
  } else if (S.nl > 0) {
    MGRX_CK(cudaMemsetAsync(z, 0, sizeof(double) * S.nl, c.s));
  }
  S.f_relax.apply(r, S.Floc.get(), S.zF.get(), nullptr, c);
  if (S.nf > 0) {
    k_scatter_add_s<<<blocks_for(S.nf, 256), 256, 0, c.s>>>(S.nf, S.Floc.get(), S.zF.get(), z);
    MGRX_LAUNCH_CK();
    count_launch();
  }
  halo(S.A, z, c);
  spmv_residual(S.A.M, z, v, nullptr, S.t.get(), c.s);
  halo(S.R, S.t.get(), c);
  spmv(S.R.M, S.t.get(), S.rc.get(), c.s);
  apply_level(l + 1, S.rc.get(), S.e.get());
  halo(S.P, S.e.get(), c);
  spmv_add(S.P.M, S.e.get(), z, c.s);
}

void Shard::prec(const double* v, double* z) {
  static const bool graphs = [] {
    const char* e = std::getenv("MGRX_GRAPHS");
    return !(e && e[0] == '0');
  }();
  if (!graphs || !comm->graph_safe()) {
    apply_level(0, v, z);
    return;
  }
  if (!graph || graph_in != v || graph_out != z) {
    if (graph) cudaGraphExecDestroy(graph);
    graph = nullptr;
    cudaGraph_t g;
    MGRX_CK(cudaStreamBeginCapture(c.s, cudaStreamCaptureModeThreadLocal));
    const long long before = g_launches;
    apply_level(0, v, z);
    graph_nodes_ = g_launches - before;
    MGRX_CK(cudaStreamEndCapture(c.s, &g));
    MGRX_CK(cudaGraphInstantiate(&graph, g, 0));
    cudaGraphDestroy(g);
    graph_in = v;
    graph_out = z;
    g_launches = before;
  }
  MGRX_CK(cudaGraphLaunch(graph, c.s));
  count_launch(graph_nodes_);
}

void Shard::apply(const double* v, double* z) {
  const int n = spaces.front().own;
  // z may lack halo room: run into zext and copy out
  prec(v, zext.get());
  d2d(z, zext.get(), n, c.s);
  MGRX_CK(cudaStreamSynchronize(c.s));
}

// Right-preconditioned restarted GMRES (proj/src/krylov.cpp:37-147) over the
// slabs: the control flow of gmres_device's per-projection MGS path, with
// every inner product reduced across ranks (all-gather + rank-order sum).
GmresResult Shard::solve(const double* b, double* x, const KrylovSpec& cfg) {
  const int n = spaces.front().own;
  cudaStream_t s = c.s;
  if (cfg.restart < 1) throw InvalidArgument("gmres: restart must be >= 1");
  const int m = cfg.restart;
  ws.ensure(n, m, s);
  double* S = ws.scal.get();
  double* s_n0 = S;
  double* s_n1 = S + 1;
  double* s_hp = S + 2;
  double* s_hc = S + 3 + (m + 1);
  double* H_pin = ws.hpinned;
  const size_t col_bytes = sizeof(double) * (3 + 2 * (m + 1) + 1);
  double* L = loc.get();
  auto reduce = [&](double* dh, double* hacc, bool acc, double* dn) {
    c.comm->allgather(L, gbuf.get(), 2, s);
    k_fold2<<<1, 1, 0, s>>>(c.size, gbuf.get(), dh, hacc, acc ? 1 : 0, dn);
    MGRX_LAUNCH_CK();
    count_launch();
  };
  auto norm2 = [&](const double* v) {
    mgs_step(n, const_cast<double*>(v), nullptr, nullptr, nullptr, true, ws, nullptr, nullptr, false, L + 1, s);
    reduce(nullptr, nullptr, false, s_n0);
    return read_scalar(s_n0, s);
  };
  double* xe = xext.get();
  d2d(xe, x, n, s);
  GmresResult res;
  const double bb = norm2(b);
  if (!std::isfinite(bb)) throw RuntimeError("gmres: rhs contains non-finite entries");
  const double bnorm = std::sqrt(bb);
  if (bnorm == 0.0) {
    if (n > 0) MGRX_CK(cudaMemsetAsync(x, 0, sizeof(double) * n, s));
    MGRX_CK(cudaStreamSynchronize(s));
    res.converged = true;
    return res;
  }
  const double target = std::max(cfg.rel_tol * bnorm, cfg.abs_tol);
  std::vector<double> Hm(static_cast<size_t>(m + 1) * m, 0.0), cs(m, 0.0), sn(m, 0.0), g(m + 1, 0.0);
  auto h = [&](int i, int j) -> double& { return Hm[static_cast<size_t>(j) * (m + 1) + i]; };
  double* V = ws.V.get();
  auto col = [&](int j) { return V + static_cast<size_t>(j) * n; };
  auto finish = [&] {
    d2d(x, xe, n, s);
    MGRX_CK(cudaStreamSynchronize(s));
  };
  auto mgs_pass = [&](int k, bool second) {
    for (int i = 0; i <= k; ++i) {
      mgs_step(n, ws.w.get(), i ? col(i - 1) : nullptr, i ? s_hp + (i - 1) : nullptr, col(i), i == 0 && !second,
               ws, L, nullptr, false, (i == 0 && !second) ? L + 1 : nullptr, s);
      reduce(s_hp + i, s_hc + i, second, (i == 0 && !second) ? s_n0 : nullptr);
    }
    mgs_step(n, ws.w.get(), col(k), s_hp + k, nullptr, true, ws, nullptr, nullptr, false, L + 1, s);
    reduce(nullptr, nullptr, false, s_n1);
    MGRX_CK(cudaMemcpyAsync(H_pin, S, col_bytes, cudaMemcpyDeviceToHost, s));
    MGRX_CK(cudaStreamSynchronize(s));
  };

  while (res.iterations < cfg.max_iters) {
    halo(Afine, xe, c);
    spmv_residual(Afine.M, xe, b, nullptr, ws.r.get(), s);  // r = b - A x
    const double rnorm = std::sqrt(norm2(ws.r.get()));
    if (!std::isfinite(rnorm)) throw RuntimeError("gmres: residual is non-finite");
    if (rnorm <= target) {
      res.converged = true;
      res.final_residual = rnorm / bnorm;
      res.history.push_back(res.final_residual);
      finish();
      return res;
    }
    vec_scale(n, ws.r.get(), rnorm, col(0), s);
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = rnorm;
    int k = 0;
    bool breakdown = false;
    for (; k < m && res.iterations < cfg.max_iters; ++k) {
      prec(col(k), zext.get());
      halo(Afine, zext.get(), c);
      spmv(Afine.M, zext.get(), ws.w.get(), s);  // w = A M^{-1} v_k
      double wn;
      if (fused) {
        // both MGS passes, the re-orthogonalisation test and v_{k+1} in one
        // kernel per rank, partials exchanged through the peers' mailboxes
        if (c.size == 1) {
          MGRX_CK(cudaMemsetAsync(S + m + 3, 0, sizeof(double), s));
          arnoldi_probe(n, k, 0, ws, s);
        } else {
          arnoldi_sharded(n, k, 0, peers_arg(), ws, s);
        }
        MGRX_CK(cudaMemcpyAsync(H_pin, S, col_bytes, cudaMemcpyDeviceToHost, s));
        MGRX_CK(cudaStreamSynchronize(s));
        if (H_pin[m + 3] != 0.0) throw RuntimeError("sharded Arnoldi: a peer did not answer (exchange timed out)");
        wn = std::sqrt(H_pin[1]);
      } else {
        // pass 1: h_i = v_i . w ; w -= h_i v_i  (krylov.cpp:84-89)
        mgs_pass(k, false);
        const double w0 = std::sqrt(H_pin[0]);
        wn = std::sqrt(H_pin[1]);
        if (wn < w0 / std::sqrt(2.0)) {
          mgs_pass(k, true);  // pass 2 (krylov.cpp:90-96): H(i,k) += h_i
          wn = std::sqrt(H_pin[1]);
        }
        if (!(wn < 1e-300)) vec_scale(n, ws.w.get(), wn, col(k + 1), s);
      }
      const double* hc = H_pin + 3 + (m + 1);
      for (int i = 0; i <= k; ++i) h(i, k) = hc[i];
      h(k + 1, k) = wn;
      if (!std::isfinite(wn)) throw RuntimeError("gmres: Arnoldi vector is non-finite");
      const bool happy = wn < 1e-300;
      for (int i = 0; i < k; ++i) {  // Givens (krylov.cpp:11-33)
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
      basis_combine(n, keff, V, s_hp, ws.u.get(), s);
      prec(ws.u.get(), zext.get());
      vec_add(n, zext.get(), xe, s);  // x += M^{-1}(V y)
      MGRX_CK(cudaStreamSynchronize(s));
    }
    halo(Afine, xe, c);
    spmv_residual(Afine.M, xe, b, nullptr, ws.r.get(), s);
    const double tn = std::sqrt(norm2(ws.r.get()));
    if (!std::isfinite(tn)) throw RuntimeError("gmres: residual is non-finite");
    res.history.push_back(tn / bnorm);
    if (tn <= target) {
      res.converged = true;
      res.final_residual = tn / bnorm;
      finish();
      return res;
    }
    if (breakdown) throw RuntimeError("gmres: Arnoldi breakdown before reaching tolerance");
    res.final_residual = tn / bnorm;
  }
  finish();
  return res;
}

}  // namespace mgrx
