// Shard setup as PLANS ("build on GPU 0 ... then scatter").
//
// A plan is the byte stream from which one rank materialises its shard: for
// every operator of every level, the rank's row slab (local CSR with columns
// renumbered [owned | halo]) with its halo recv / send lists; the index-space
// partitions; the local F / C rows of each MGR level; Jacobi diagonals; and,
// for the small replicated parts (dense coarse solves, the replicated coarse
// AMG levels), the global small matrix, which every rank then factors or
// coarsens itself with the same bit-exact setup kernels.
//
// Planner (host, on the rank that holds the global hierarchy) writes the
// plans of ALL ranks in one traversal (each global operator is downloaded
// once and cut for every rank: halos first, then every rank's send lists
// from its neighbours' halos). Loader (every rank) reads its plan in the same
// traversal order and builds the device structures.
//
// Two ways to get a plan:
//  * Shard::build: every rank holds a replica of the global hierarchy and
//    plans for itself (phase 1, no setup traffic);
//  * Shard::build_scatter: only the root holds the global hierarchy; it
//    plans for every rank and ships each rank its plan over the comm (NCCL
//    send/recv, or device copies in a local group). The other ranks never
//    hold a global operator: per-rank device memory is the slab (plus the
//    small replicated coarse parts), and the root may free its hierarchy as
//    soon as the shards exist.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>

#include "shard.cuh"

namespace mgrx {

// ---------------------------------------------------------------------------
// byte streams
class PlanW {
 public:
  std::vector<unsigned char> b;
  void raw(const void* p, size_t n) {
    const auto* c = static_cast<const unsigned char*>(p);
    b.insert(b.end(), c, c + n);
  }
  void i32(int v) { raw(&v, sizeof v); }
  void f64(double v) { raw(&v, sizeof v); }
  template <class T>
  void vec(const T* p, size_t n) {
    const long long k = static_cast<long long>(n);
    raw(&k, sizeof k);
    if (n) raw(p, n * sizeof(T));
  }
  template <class T>
  void vec(const std::vector<T>& v) {
    vec(v.data(), v.size());
  }
  void str(const std::string& s) { vec(s.data(), s.size()); }
};

class PlanR {
 public:
  PlanR(const unsigned char* p, size_t n) : p_(p), n_(n) {}
  void raw(void* d, size_t n) {
    if (off_ + n > n_) throw RuntimeError("sharded setup: truncated plan");
    std::memcpy(d, p_ + off_, n);
    off_ += n;
  }
  int i32() {
    int v;
    raw(&v, sizeof v);
    return v;
  }
  double f64() {
    double v;
    raw(&v, sizeof v);
    return v;
  }
  template <class T>
  std::vector<T> vec() {
    long long k;
    raw(&k, sizeof k);
    if (k < 0) throw RuntimeError("sharded setup: corrupt plan");
    std::vector<T> v(static_cast<size_t>(k));
    if (k) raw(v.data(), static_cast<size_t>(k) * sizeof(T));
    return v;
  }
  std::string str() {
    const std::vector<char> c = vec<char>();
    return std::string(c.begin(), c.end());
  }
  bool done() const { return off_ == n_; }

 private:
  const unsigned char* p_;
  size_t n_, off_ = 0;
};

namespace {

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

DVec<int> upload_ints(const std::vector<int>& v, cudaStream_t s) {
  DVec<int> d(v.size() > 0 ? v.size() : 1, s);
  d.upload(v.data(), v.size());
  return d;
}

void alloc_cap(DVec<double>& v, const Space& sp, cudaStream_t s) { v.alloc(sp.cap > 0 ? sp.cap : 1, s); }

// One rank's slab of an operator (rows of `rows` owned by the rank, columns
// of `cols` renumbered [owned | halo]; entries keep their order, so every
// row sum is the single-GPU one). recv / send: (peer, offset, count) triples.
struct OpSlab {
  int own = 0, nhalo = 0;
  std::vector<int> lp, lc, recv, send, sidx;
  std::vector<double> lv;
};

// Slabs of every rank in one pass: each rank's halo is the sorted set of
// non-owned columns its rows read; the send list of rank q to rank p is the
// part of p's halo that q owns.
std::vector<OpSlab> cut_op(const HostCsr& G, const Part& rows, const Part& cols) {
  const int size = static_cast<int>(rows.st.size()) - 1;
  if (G.rows != rows.total() || G.cols != cols.total())
    throw RuntimeError("sharded solve: operator does not match its index spaces");
  std::vector<OpSlab> out(size);
  std::vector<std::vector<int>> halo(size);
  for (int q = 0; q < size; ++q) {
    OpSlab& o = out[q];
    const int r0 = rows.lo(q), r1 = rows.hi(q), c0 = cols.lo(q), c1 = cols.hi(q);
    std::vector<int>& h = halo[q];
    for (int k = G.ptr[r0]; k < G.ptr[r1]; ++k)
      if (G.col[k] < c0 || G.col[k] >= c1) h.push_back(G.col[k]);
    std::sort(h.begin(), h.end());
    h.erase(std::unique(h.begin(), h.end()), h.end());
    o.own = c1 - c0;
    o.nhalo = static_cast<int>(h.size());
    const int m = r1 - r0;
    o.lp.resize(m + 1);
    for (int i = 0; i <= m; ++i) o.lp[i] = G.ptr[r0 + i] - G.ptr[r0];
    o.lc.resize(G.ptr[r1] - G.ptr[r0]);
    o.lv.assign(G.val.begin() + G.ptr[r0], G.val.begin() + G.ptr[r1]);
    for (int k = G.ptr[r0]; k < G.ptr[r1]; ++k) {
      const int j = G.col[k];
      o.lc[k - G.ptr[r0]] = (j >= c0 && j < c1)
                                ? j - c0
                                : o.own + static_cast<int>(std::lower_bound(h.begin(), h.end(), j) - h.begin());
    }
    for (int a = 0; a < o.nhalo;) {  // recv segments: halo grouped by owner (monotone in j)
      const int p = cols.owner(h[a]);
      int b = a;
      while (b < o.nhalo && h[b] < cols.hi(p)) ++b;
      o.recv.insert(o.recv.end(), {p, a, b - a});
      a = b;
    }
  }
  for (int q = 0; q < size; ++q) {
    OpSlab& o = out[q];
    const int c0 = cols.lo(q), c1 = cols.hi(q);
    for (int p = 0; p < size; ++p) {
      if (p == q) continue;
      const std::vector<int>& h = halo[p];
      const auto lo = std::lower_bound(h.begin(), h.end(), c0), hi = std::lower_bound(h.begin(), h.end(), c1);
      if (lo == hi) continue;
      o.send.insert(o.send.end(), {p, static_cast<int>(o.sidx.size()), static_cast<int>(hi - lo)});
      for (auto it = lo; it != hi; ++it) o.sidx.push_back(*it - c0);
    }
  }
  return out;
}

int repl_rows_env() {
  static const int m = [] {
    const char* v = std::getenv("MGRX_SHARD_REPL_ROWS");
    return v ? std::atoi(v) : 65536;
  }();
  return m;
}

// First AMG level that the sharded V-cycle replicates: small, Jacobi-type
// smoothing from there on (the single-GPU smoother path without a gather),
// more than one rank; -1: none.
int replicate_from(const AmgHier& g, int size) {
  const int nl = static_cast<int>(g.levels.size());
  if (size <= 1 || repl_rows_env() <= 0) return -1;
  for (int l = 1; l < nl; ++l) {
    if (g.levels[l].A.rows > repl_rows_env()) continue;
    bool ok = true;
    for (int k = l; k < nl - 1 && ok; ++k) {
      const BoundRelax* bs[2] = {&g.levels[k].pre, &g.levels[k].post};
      for (const BoundRelax* b : bs)
        ok = ok && (b->spec.kind == Smoother::jacobi || b->spec.kind == Smoother::l1_jacobi) &&
             (b->spec.sweeps <= 1 || b->n <= fold_sweep0_max_rows());
    }
    if (ok) return l;
  }
  return -1;
}

void write_smoother(PlanW& w, const SmootherSpec& s) {
  w.i32(static_cast<int>(s.kind));
  w.i32(s.sweeps);
  w.f64(s.weight);
}
SmootherSpec read_smoother(PlanR& r) {
  SmootherSpec s;
  s.kind = static_cast<Smoother>(r.i32());
  s.sweeps = r.i32();
  s.weight = r.f64();
  return s;
}

// ---------------------------------------------------------------------------
// Planner: every rank's plan from the global hierarchy
struct Planner {
  const MgrHier& h;
  const DCsr& A;
  Part fine;
  int size;
  cudaStream_t s;
  std::vector<PlanW> W;
  std::map<const DCsr*, HostCsr> mats;

  Planner(const MgrHier& hh, const DCsr& AA, const Part& p, cudaStream_t st)
      : h(hh), A(AA), fine(p), size(static_cast<int>(p.st.size()) - 1), s(st), W(size) {}

  const HostCsr& host(const DCsr& M) {
    auto it = mats.find(&M);
    if (it != mats.end()) return it->second;
    return mats.emplace(&M, to_host(M, s)).first->second;
  }
  void part_all(const Part& p) {
    for (PlanW& w : W) w.vec(p.st);
  }
  void op(const DCsr& G, const Part& rows, const Part& cols) {
    std::vector<OpSlab> sl = cut_op(host(G), rows, cols);
    for (int q = 0; q < size; ++q) {
      PlanW& w = W[q];
      const OpSlab& o = sl[q];
      w.i32(o.own);
      w.i32(o.nhalo);
      w.vec(o.lp);
      w.vec(o.lc);
      w.vec(o.lv);
      w.vec(o.recv);
      w.vec(o.send);
      w.vec(o.sidx);
    }
  }
  // the whole (small) matrix to every rank
  void full(const DCsr& G) {
    const HostCsr& c = host(G);
    for (PlanW& w : W) {
      w.i32(c.rows);
      w.i32(c.cols);
      w.vec(c.ptr);
      w.vec(c.col);
      w.vec(c.val);
    }
  }
  void relax(const BoundRelax& g, const DCsr& Ag, const Part& space) {
    for (PlanW& w : W) write_smoother(w, g.spec);
    switch (g.spec.kind) {
      case Smoother::jacobi:
      case Smoother::l1_jacobi: {
        const std::vector<double> d = dl(g.dinv, space.total(), s);
        for (int q = 0; q < size; ++q) W[q].vec(d.data() + space.lo(q), static_cast<size_t>(space.n(q)));
        if (g.spec.sweeps > 1) op(Ag, space, space);
        break;
      }
      case Smoother::amg_vcycle:
        amg(*g.amg, space);
        if (g.spec.sweeps > 1) op(Ag, space, space);
        break;
      case Smoother::dense_lu:
        full(Ag);
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
  void amg(const AmgHier& g, const Part& fine_sp) {
    const int nl = static_cast<int>(g.levels.size());
    for (PlanW& w : W) w.i32(nl);
    std::vector<Part> sp(nl);
    sp[0] = fine_sp;
    for (int l = 1; l < nl; ++l) {
      const AmgLevelD& G = g.levels[l - 1];
      sp[l] = sub_part(sp[l - 1], dl(G.C, G.P.cols, s));
      part_all(sp[l]);
    }
    const int from = replicate_from(g, size);
    for (PlanW& w : W) w.i32(from);
    for (int l = 0; l < nl; ++l) {
      if (l == from) {
        // replicated levels: the level's global matrix, its unknown map and
        // the AMG configuration; every rank coarsens it (bit-exact setup)
        full(g.levels[l].A);
        for (PlanW& w : W) {
          w.vec(g.levels[l].umap);
          w.f64(g.spec.strength_theta);
          w.i32(g.spec.max_levels - l);
          w.i32(g.spec.coarse_size);
          write_smoother(w, g.spec.pre);
          write_smoother(w, g.spec.post);
        }
        return;
      }
      if (l == nl - 1) {
        full(g.levels[l].A);  // coarsest: every rank factors it
        return;
      }
      const AmgLevelD& G = g.levels[l];
      op(G.A, sp[l], sp[l]);
      op(G.R, sp[l + 1], sp[l]);
      op(G.P, sp[l], sp[l + 1]);
      relax(G.pre, G.A, sp[l]);
      relax(G.post, G.A, sp[l]);
    }
  }
  void all() {
    part_all(fine);
    for (PlanW& w : W) w.i32(static_cast<int>(h.levels.size()));
    Part cur = fine;
    for (const MgrLevelD& G : h.levels) {
      const std::vector<int> F = dl(G.F, G.F.size(), s);
      const std::vector<int> C = dl(G.C, G.C.size(), s);
      const Part sf = sub_part(cur, F), sc = sub_part(cur, C);
      part_all(sf);
      part_all(sc);
      for (int q = 0; q < size; ++q) {
        const int lo = cur.lo(q);
        std::vector<int> fl(sf.n(q)), cl(sc.n(q));
        for (int i = 0; i < sf.n(q); ++i) fl[i] = F[sf.lo(q) + i] - lo;
        for (int i = 0; i < sc.n(q); ++i) cl[i] = C[sc.lo(q) + i] - lo;
        W[q].vec(fl);
        W[q].vec(cl);
      }
      const bool general = !G.injection || G.g_relax.has_value();
      for (PlanW& w : W) {
        w.i32(G.injection ? 1 : 0);
        w.i32(general ? 1 : 0);
        w.i32(G.g_relax.has_value() ? 1 : 0);
      }
      op(G.P, cur, sc);
      if (general) {
        op(G.A, cur, cur);
        op(G.R, sc, cur);
        if (G.g_relax) relax(*G.g_relax, G.A, cur);
      } else {
        op(G.Acf, sc, sf);
      }
      relax(G.f_relax, G.Aff, sf);
      cur = sc;
    }
    const bool dense = h.coarse_spec.kind == Coarse::dense_lu;
    for (PlanW& w : W) w.i32(dense ? 0 : 1);
    if (dense) {
      full(h.A_coarse);
    } else {
      amg(*h.coarse_amg, cur);
      for (PlanW& w : W) w.i32(h.coarse_spec.cycles);
      if (h.coarse_spec.cycles > 1) op(h.A_coarse, cur, cur);
    }
    op(A, fine, fine);
    for (PlanW& w : W) w.i32(0x5eed);  // end marker
  }
};

// ---------------------------------------------------------------------------
// Loader: one rank's shard from its plan
struct Loader {
  PlanR& R;
  Shard& sh;
  ShardCtx& c;

  Part part() {
    Part p;
    p.st = R.vec<int>();
    if (static_cast<int>(p.st.size()) != c.size + 1) throw RuntimeError("sharded setup: plan is for another group");
    return p;
  }
  void op(SOp& o, Space& cols) {
    o.own = R.i32();
    o.nhalo = R.i32();
    const std::vector<int> lp = R.vec<int>(), lc = R.vec<int>();
    const std::vector<double> lv = R.vec<double>();
    const std::vector<int> recv = R.vec<int>(), send = R.vec<int>(), sidx = R.vec<int>();
    cols.need(o.nhalo);
    const int m = static_cast<int>(lp.size()) - 1;
    cudaStream_t s = c.s;
    o.M = DCsr();
    o.M.rows = m;
    o.M.cols = o.own + o.nhalo;
    o.M.nnz = static_cast<int>(lc.size());
    o.M.ptr.alloc(m + 1, s);
    o.M.ptr.upload(lp.data(), m + 1);
    o.M.col.alloc(lc.size() > 0 ? lc.size() : 1, s);
    o.M.col.upload(lc.data(), lc.size());
    o.M.val.alloc(lv.size() > 0 ? lv.size() : 1, s);
    o.M.val.upload(lv.data(), lv.size());
    o.recv.clear();
    o.send.clear();
    for (size_t i = 0; i + 2 < recv.size(); i += 3) o.recv.push_back({recv[i], recv[i + 1], recv[i + 2]});
    for (size_t i = 0; i + 2 < send.size(); i += 3) o.send.push_back({send[i], send[i + 1], send[i + 2]});
    o.sidx = upload_ints(sidx, s);
    o.sbuf.alloc(sidx.size() > 0 ? sidx.size() : 1, s);
    o.built = true;
    spmv_prepare(o.M, s);
  }
  DCsr& full() {
    const int rows = R.i32(), cols = R.i32();
    const std::vector<int> ptr = R.vec<int>(), col = R.vec<int>();
    const std::vector<double> val = R.vec<double>();
    sh.own_mat.emplace_back();
    DCsr& M = sh.own_mat.back();
    M.rows = rows;
    M.cols = cols;
    M.nnz = static_cast<int>(col.size());
    M.ptr.alloc(rows + 1, c.s);
    M.ptr.upload(ptr.data(), ptr.size());
    M.col.alloc(col.size() > 0 ? col.size() : 1, c.s);
    M.col.upload(col.data(), col.size());
    M.val.alloc(val.size() > 0 ? val.size() : 1, c.s);
    M.val.upload(val.data(), val.size());
    return M;
  }
  // factor a replicated small matrix (the same dense_factor call as the
  // global setup: bitwise the same factors)
  const DenseLU* factor(const DCsr& M) {
    sh.own_lu.emplace_back();
    dense_factor(M, sh.own_lu.back(), c.s);
    return &sh.own_lu.back();
  }
  void relax(SRelax& x, Space& space) {
    const SmootherSpec sp = read_smoother(R);
    x.kind = sp.kind;
    x.sweeps = sp.sweeps;
    x.weight = sp.weight;
    x.sp = &space;
    x.n = space.own;
    switch (x.kind) {
      case Smoother::jacobi:
      case Smoother::l1_jacobi: {
        const std::vector<double> d = R.vec<double>();
        x.dinv.alloc(x.n > 0 ? x.n : 1, c.s);
        x.dinv.upload(d.data(), d.size());
        if (x.sweeps > 1) op(x.A, space);
        break;
      }
      case Smoother::amg_vcycle:
        x.amg = std::make_unique<SAmg>();
        amg(*x.amg, space);
        if (x.sweeps > 1) op(x.A, space);
        break;
      case Smoother::dense_lu:
        x.dense.build(factor(full()), space.part, c.s);
        break;
      default:
        throw RuntimeError("sharded setup: smoother kind not supported across slabs");
    }
  }
  void amg(SAmg& a, Space& fine) {
    const int nl = R.i32();
    std::vector<Space*> sp(nl);
    sp[0] = &fine;
    for (int l = 1; l < nl; ++l) {
      a.spaces.push_back(make_space(part(), c.rank));
      sp[l] = &a.spaces.back();
    }
    const int from = R.i32();
    for (int l = 0; l < nl; ++l) {
      a.L.emplace_back();
      SAmgLevel& S = a.L.back();
      S.sp = sp[l];
      if (l == from) {
        DCsr& M = full();
        const std::vector<int> um = R.vec<int>();
        AmgSpec cfg;
        cfg.strength_theta = R.f64();
        cfg.max_levels = R.i32();
        cfg.coarse_size = R.i32();
        cfg.pre = read_smoother(R);
        cfg.post = read_smoother(R);
        sh.own_amg.push_back(std::make_unique<AmgHier>());
        AmgHier& sub = *sh.own_amg.back();
        sub.setup(M, cfg, um, c.s);
        prepare_amg(sub, c.s);
        a.rep.build(sub, 0, sp[l]->part, c.s);
        a.rep.at = l;
        return;
      }
      if (l == nl - 1) {
        a.coarse.build(factor(full()), sp[l]->part, c.s);
        return;
      }
      op(S.A, *sp[l]);
      op(S.R, *sp[l]);
      op(S.P, *sp[l + 1]);
      relax(S.pre, *sp[l]);
      relax(S.post, *sp[l]);
    }
  }
  void all() {
    sh.spaces.push_back(make_space(part(), c.rank));
    Space* cur = &sh.spaces.back();
    sh.row_begin = cur->part.lo(c.rank);
    sh.row_end = cur->part.hi(c.rank);
    const int nlev = R.i32();
    for (int l = 0; l < nlev; ++l) {
      sh.levels.emplace_back();
      SMgrLevel& S = sh.levels.back();
      S.sl = cur;
      sh.spaces.push_back(make_space(part(), c.rank));
      S.sf = &sh.spaces.back();
      sh.spaces.push_back(make_space(part(), c.rank));
      S.sc = &sh.spaces.back();
      S.nl = cur->own;
      S.nf = S.sf->own;
      S.nc = S.sc->own;
      const std::vector<int> fl = R.vec<int>(), cl = R.vec<int>();
      std::vector<int> fp(S.nl, -1);
      for (int i = 0; i < S.nf; ++i) fp[fl[i]] = i;
      S.Floc = upload_ints(fl, c.s);
      S.Cloc = upload_ints(cl, c.s);
      S.fpos = upload_ints(fp, c.s);
      S.injection = R.i32() != 0;
      S.general = R.i32() != 0;
      const bool has_g = R.i32() != 0;
      op(S.P, *S.sc);
      if (S.general) {
        op(S.A, *cur);
        op(S.R, *cur);
        if (has_g) {
          S.g_relax = std::make_unique<SRelax>();
          relax(*S.g_relax, *cur);
        }
      } else {
        op(S.Acf, *S.sf);
      }
      relax(S.f_relax, *S.sf);
      cur = S.sc;
    }
    if (R.i32() == 0) {
      sh.coarse_lu.build(factor(full()), cur->part, c.s);
    } else {
      sh.coarse_amg = std::make_unique<SAmg>();
      amg(*sh.coarse_amg, *cur);
      sh.coarse_cycles = R.i32();
      if (sh.coarse_cycles > 1) op(sh.Acoarse, *cur);
    }
    op(sh.Afine, sh.spaces.front());
    if (R.i32() != 0x5eed || !R.done()) throw RuntimeError("sharded setup: plan / loader mismatch");
  }
};

Part check_starts(const std::vector<int>& st, int size, int n) {
  Part p;
  p.st = st;
  if (static_cast<int>(p.st.size()) != size + 1 || p.st.front() != 0 || (n >= 0 && p.st.back() != n))
    throw InvalidArgument("sharded solve: row starts must be size+1 offsets from 0 to n");
  for (int q = 0; q < size; ++q)
    if (p.st[q + 1] <= p.st[q]) throw InvalidArgument("sharded solve: every rank needs at least one row");
  return p;
}

}  // namespace

void Shard::load(const std::vector<unsigned char>& plan) {
  PlanR R(plan.data(), plan.size());
  Loader ld{R, *this, c};
  ld.all();
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
  const Space* last = levels.empty() ? &spaces.front() : levels.back().sc;
  if (coarse_amg) coarse_amg->alloc(c.s);
  alloc_cap(ct, *last, c.s);
  alloc_cap(cd, *last, c.s);
  alloc_cap(xext, spaces.front(), c.s);
  alloc_cap(zext, spaces.front(), c.s);
  loc.alloc(2, c.s);
  loc.zero();
  gbuf.alloc(2 * c.size, c.s);
  MGRX_CK(cudaStreamSynchronize(c.s));
}

std::vector<std::vector<unsigned char>> shard_plans(const MgrHier& h, const DCsr& A, const std::vector<int>& starts,
                                                    cudaStream_t s) {
  Planner p(h, A, check_starts(starts, static_cast<int>(starts.size()) - 1, A.rows), s);
  p.all();
  std::vector<std::vector<unsigned char>> out(p.W.size());
  for (size_t q = 0; q < p.W.size(); ++q) out[q] = std::move(p.W[q].b);
  return out;
}

void Shard::build(MgrHier& h, const DCsr& A, const std::vector<int>& fine_starts, std::unique_ptr<Comm> cm,
                  cudaStream_t stream) {
  comm = std::move(cm);
  c.comm = comm.get();
  c.rank = comm->rank;
  c.size = comm->size;
  c.s = stream;
  check_starts(fine_starts, c.size, A.rows);
  // every rank holds the global hierarchy: plan for all, keep this rank's
  std::vector<std::vector<unsigned char>> plans = shard_plans(h, A, fine_starts, stream);
  load(plans[c.rank]);
  setup_fused();
}

// Root (rank 0, holding the global hierarchy) plans for every rank and sends
// each its plan: a byte count, then the bytes (as doubles) over the comm's
// point-to-point exchange. A planning error reaches every rank as its plan
// (status 0 + message), so no rank waits for a plan that never comes.
void Shard::build_scatter(MgrHier* h, const DCsr* A, const std::vector<int>& fine_starts, std::unique_ptr<Comm> cm,
                          cudaStream_t stream) {
  comm = std::move(cm);
  c.comm = comm.get();
  c.rank = comm->rank;
  c.size = comm->size;
  c.s = stream;
  const bool root = c.rank == 0;
  if (root != (h != nullptr && A != nullptr))
    throw InvalidArgument("mgrx_shard_create_scatter: rank 0 (and only rank 0) passes the global hierarchy");
  check_starts(fine_starts, c.size, root ? A->rows : -1);
  std::vector<std::vector<unsigned char>> plans;
  if (root) {
    try {
      plans = shard_plans(*h, *A, fine_starts, stream);
      for (auto& p : plans) p.insert(p.begin(), 1);  // status ok
    } catch (const std::exception& e) {
      plans.assign(c.size, {0});
      const std::string m = e.what();
      for (auto& p : plans) p.insert(p.end(), m.begin(), m.end());
    }
  }
  // sizes
  DVec<double> nb(c.size, stream);
  std::vector<double> hn(c.size, 0.0);
  if (root)
    for (int q = 0; q < c.size; ++q) hn[q] = static_cast<double>(plans[q].size());
  nb.upload(hn.data(), c.size);
  {
    std::vector<Xfer> sends, recvs;
    if (root)
      for (int q = 1; q < c.size; ++q) sends.push_back({q, nb.get() + q, 1});
    else
      recvs.push_back({0, nb.get() + c.rank, 1});
    if (c.size > 1) c.comm->exchange(sends, recvs, stream);
  }
  const size_t mine = static_cast<size_t>(nb.download(c.size)[c.rank]);
  // payloads
  std::vector<unsigned char> plan;
  if (root) {
    std::vector<DVec<double>> bufs(c.size);
    std::vector<Xfer> sends;
    for (int q = 1; q < c.size; ++q) {
      const size_t nd = (plans[q].size() + 7) / 8;
      bufs[q].alloc(nd > 0 ? nd : 1, stream);
      MGRX_CK(cudaMemcpyAsync(bufs[q].get(), plans[q].data(), plans[q].size(), cudaMemcpyHostToDevice, stream));
      sends.push_back({q, bufs[q].get(), static_cast<int>(nd)});
    }
    if (!sends.empty()) c.comm->exchange(sends, {}, stream);
    MGRX_CK(cudaStreamSynchronize(stream));
    plan = std::move(plans[0]);
  } else {
    const size_t nd = (mine + 7) / 8;
    DVec<double> buf(nd > 0 ? nd : 1, stream);
    c.comm->exchange({}, {{0, buf.get(), static_cast<int>(nd)}}, stream);
    plan.resize(mine);
    MGRX_CK(cudaMemcpyAsync(plan.data(), buf.get(), mine, cudaMemcpyDeviceToHost, stream));
    MGRX_CK(cudaStreamSynchronize(stream));
  }
  if (plan.empty() || plan[0] != 1)
    throw RuntimeError(plan.size() > 1 ? std::string(plan.begin() + 1, plan.end()) : "sharded setup: no plan");
  plan.erase(plan.begin());
  load(plan);
  setup_fused();
}

}  // namespace mgrx
