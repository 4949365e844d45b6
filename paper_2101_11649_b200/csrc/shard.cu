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
  dense_solve(*lu, full.get(), sol.get(), c.s, c.exact);
  d2d(z, sol.get() + part.lo(c.rank), own, c.s);
}

// ---------------------------------------------------------------------------
// smoothers
// ---------------------------------------------------------------------------
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
  at = l;
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
  if (l == rep.at) {
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
  for (auto& kv : graphs_)
    if (kv.second.first) cudaGraphExecDestroy(kv.second.first);
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
  // one captured graph per (input, output, dense mode): the solve alternates
  // M^-1 U (every step) and M^-1 (V y) (once per cycle)
  const auto key = std::make_tuple(v, z, c.exact);
  auto it = graphs_.find(key);
  if (it == graphs_.end()) {
    cudaGraph_t g;
    cudaGraphExec_t ex = nullptr;
    MGRX_CK(cudaStreamBeginCapture(c.s, cudaStreamCaptureModeThreadLocal));
    const long long before = g_launches;
    apply_level(0, v, z);
    const long long nodes = g_launches - before;
    MGRX_CK(cudaStreamEndCapture(c.s, &g));
    MGRX_CK(cudaGraphInstantiate(&ex, g, 0));
    cudaGraphDestroy(g);
    g_launches = before;
    it = graphs_.emplace(key, std::make_pair(ex, nodes)).first;
  }
  MGRX_CK(cudaGraphLaunch(it->second.first, c.s));
  count_launch(it->second.second);
}

void Shard::apply(const double* v, double* z) {
  c.exact = true;
  const int n = spaces.front().own;
  // z may lack halo room: run into zext and copy out
  prec(v, zext.get());
  d2d(z, zext.get(), n, c.s);
  MGRX_CK(cudaStreamSynchronize(c.s));
}

// Right-preconditioned restarted GMRES (proj/src/krylov.cpp:37-147) over the
// slabs: the control flow of gmres_device's per-projection MGS path, with
// every inner product reduced across ranks (all-gather + rank-order sum).
// Low-synchronisation variant (the default, KrylovSpec::ortho != mgs): the
// lagged CGS2 step of lowsync.cu on the slabs, its two reductions per step
// completed across ranks by an all-gather of the rank sums and a rank-order
// fold (2 collectives per step instead of 2k+4 under MGS).
GmresResult Shard::solve_lowsync(const double* b, double* x, const KrylovSpec& cfg) {
  const int n = spaces.front().own;
  cudaStream_t s = c.s;
  const int m = cfg.restart;
  c.exact = false;  // dense blocks through their inverses (tolerance-level)
  ws.ensure(n, 1, s);
  ws.ls.ensure(n, m, s);
  LsDriver drv(ws.ls, n, m, ws.w.get());
  double* U = drv.U();
  double* L = loc.get();
  const LsDriver::Allgather ag = [this](const double* in, double* out, int count, cudaStream_t st) {
    c.comm->allgather(in, out, count, st);
  };
  auto norm2 = [&](const double* v) {
    mgs_step(n, const_cast<double*>(v), nullptr, nullptr, nullptr, true, ws, nullptr, nullptr, false, L + 1, s);
    c.comm->allgather(L, gbuf.get(), 2, s);
    fold2(c.size, gbuf.get(), nullptr, nullptr, false, ws.scal.get(), s);
    return read_scalar(ws.scal.get(), s);
  };
  double* xe = xext.get();
  d2d(xe, x, n, s);
  GmresResult res;
  auto finish = [&] {
    d2d(x, xe, n, s);
    MGRX_CK(cudaStreamSynchronize(s));
  };
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
  halo(Afine, xe, c);
  spmv_residual(Afine.M, xe, b, nullptr, U, s);  // U = r = b - A x
  double rnorm = std::sqrt(norm2(U));
  std::vector<double> y;
  while (true) {
    if (!std::isfinite(rnorm)) throw RuntimeError("gmres: residual is non-finite");
    if (rnorm <= target) {
      res.converged = true;
      res.final_residual = rnorm / bnorm;
      res.history.push_back(res.final_residual);
      finish();
      return res;
    }
    if (res.iterations >= cfg.max_iters) {
      res.final_residual = rnorm / bnorm;
      finish();
      return res;
    }
    drv.start_cycle(bnorm, target, std::min(m, cfg.max_iters - res.iterations), s);
    do {
      prec(U, zext.get());
      halo(Afine, zext.get(), c);
      spmv(Afine.M, zext.get(), ws.w.get(), s);  // w = A M^{-1} U
      drv.step_sharded(c.size, ag, s);
    } while (!(drv.sync_state(s).flags & kLsCycleEnd));
    const LsState hs = drv.end_cycle(res.history, y, s);
    if (hs.flags & kLsNonFinite) throw RuntimeError("gmres: Arnoldi vector is non-finite");
    res.iterations += hs.steps;
    if (!y.empty()) {
      drv.combine(y, ws.u.get(), s);
      prec(ws.u.get(), zext.get());
      vec_add(n, zext.get(), xe, s);  // x += M^{-1}(V y)
    }
    halo(Afine, xe, c);
    spmv_residual(Afine.M, xe, b, nullptr, U, s);
    const double tn = std::sqrt(norm2(U));
    if (!std::isfinite(tn)) throw RuntimeError("gmres: residual is non-finite");
    res.history.push_back(tn / bnorm);
    if (tn <= target) {
      res.converged = true;
      res.final_residual = tn / bnorm;
      finish();
      return res;
    }
    if (hs.flags & kLsHappy) throw RuntimeError("gmres: Arnoldi breakdown before reaching tolerance");
    res.final_residual = tn / bnorm;
    if (res.iterations >= cfg.max_iters) {
      finish();
      return res;
    }
    rnorm = tn;
  }
}

GmresResult Shard::solve(const double* b, double* x, const KrylovSpec& cfg) {
  if (cfg.restart < 1) throw InvalidArgument("gmres: restart must be >= 1");
  if (cfg.ortho != kOrthoMgs && lowsync_supported(spaces.front().own, cfg.restart)) return solve_lowsync(b, x, cfg);
  c.exact = true;
  const int n = spaces.front().own;
  cudaStream_t s = c.s;
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
