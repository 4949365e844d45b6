// C-ABI boundary of libmgrx (include/mgrx.h). Maps exceptions to the
// reference's status codes and keeps the message in a thread-local string.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <functional>
#include <memory>
#include <string>

#include "../../include/mgrx.h"
#include "hierarchy.cuh"
#include "krylov.cuh"
#include "shard.cuh"

using namespace mgrx;

struct mgrx_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
};

struct mgrx_mat {
  mgrx_ctx* ctx = nullptr;
  DCsr A;
};

struct mgrx_hier {
  mgrx_ctx* ctx = nullptr;
  DCsr A;  // the hierarchy copies the fine matrix (proj/src/mgr.cpp:257)
  MgrHier H;
  GmresWork ws;
  double setup_s = 0.0;
  long long bytes = 0;     // device bytes allocated by the setup (thread counter)
  DVec<double> vin, vout;  // staging for host-pointer calls
  DVec<double> px, py, pz;  // roofline-probe operands
  DVec<char> flushbuf;      // probe: L2 flush before each timed launch
};

struct mgrx_group {
  std::shared_ptr<LocalHub> hub;  // in-process ranks (threads)
  int size = 0;
  bool host = false;              // caller-supplied host transport (one rank per process)
  HostTransport tr;
  std::unique_ptr<Comm> comm(int rank) const {
    return host ? make_host_comm(tr, rank, size) : make_local_comm(hub, rank);
  }
};

struct mgrx_shard {
  mgrx_ctx* ctx = nullptr;
  double setup_s = 0.0;    // hierarchy setup (root) + plan / scatter / load
  long long bytes = 0;     // device bytes of this rank's shard (built on this thread)
  cudaStream_t stream = nullptr;
  std::unique_ptr<Shard> sh;
  DVec<double> vin, vout;
  ~mgrx_shard() {
    sh.reset();
    vin.release();
    vout.release();
    if (stream) {
      cudaStreamSynchronize(stream);
      cudaStreamDestroy(stream);
    }
  }
};

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const std::invalid_argument*>(&e)) return MGRX_INVALID_ARGUMENT;
  return MGRX_RUNTIME;
}

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const std::exception& e) {
    return fail(e);
  } catch (...) {
    g_err = "unknown error";
    return MGRX_RUNTIME;
  }
}

void use(mgrx_ctx* c) { MGRX_CK(cudaSetDevice(c->device)); }

struct EventTimer {
  cudaEvent_t a, b;
  cudaStream_t s;
  explicit EventTimer(cudaStream_t st) : s(st) {
    MGRX_CK(cudaEventCreate(&a));
    MGRX_CK(cudaEventCreate(&b));
    MGRX_CK(cudaEventRecord(a, s));
  }
  double stop() {
    MGRX_CK(cudaEventRecord(b, s));
    MGRX_CK(cudaEventSynchronize(b));
    float ms = 0;
    MGRX_CK(cudaEventElapsedTime(&ms, a, b));
    return ms * 1e-3;
  }
  ~EventTimer() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
};

// SURVEY §8d compulsory-traffic model (bytes per launch).
double spmv_model_bytes(const DCsr& A) {
  return 12.0 * A.nnz + 4.0 * (A.rows + 1) + 8.0 * std::min<double>(A.cols, A.nnz) + 8.0 * A.rows;
}

void prepare_probe(mgrx_hier* h, const std::string& w, std::function<void()>& fn, double& bytes,
                   cudaStream_t s) {
  const size_t nmax = static_cast<size_t>(std::max(h->A.rows, h->A.cols)) + 1;
  if (h->px.size() < nmax) {
    h->px.alloc(nmax, s);
    h->py.alloc(nmax, s);
    h->pz.alloc(nmax, s);
  }
  h->px.zero();
  h->py.zero();
  h->pz.zero();
  double* x = h->px.get();
  double* y = h->py.get();
  double* z = h->pz.get();
  if (w == "mgs") {
    // fused MGS step on fine-size vectors: w -= h v_{i-1}; h_i = v_i . w
    const int n = h->A.rows;
    h->ws.ensure(n, 30, s);
    double* V = h->ws.V.get();
    double* wv = h->ws.w.get();
    MGRX_CK(cudaMemsetAsync(V, 0, sizeof(double) * 2 * static_cast<size_t>(n), s));
    MGRX_CK(cudaMemsetAsync(wv, 0, sizeof(double) * n, s));
    const double* hp = x;  // zeros
    GmresWork* ws = &h->ws;
    fn = [=] { mgs_probe(n, wv, V, hp, V + n, *ws, s); };
    bytes = 24.0 * n;  // SURVEY 8(d) MGS step model: read v_i and w, write w
    return;
  }
  if (w.rfind("arnoldi.", 0) == 0) {
    // fused Arnoldi step k on the solve's work vectors (zeros if no solve ran
    // yet), both MGS passes forced: compulsory HBM traffic is w in, each
    // v_0..v_k streamed once per pass, v_{k+1} out.
    const int n = h->A.rows;
    const int k = std::stoi(w.substr(8));
    if (h->ws.n != n || h->ws.m < 30) {
      h->ws.ensure(n, 30, s);
      MGRX_CK(cudaMemsetAsync(h->ws.V.get(), 0, sizeof(double) * static_cast<size_t>(n) * 31, s));
      MGRX_CK(cudaMemsetAsync(h->ws.w.get(), 0, sizeof(double) * n, s));
    }
    const char* e = std::getenv("MGRX_ARNOLDI_DBG");
    const int dbg = 4 | (e ? std::atoi(e) : 0);
    GmresWork* ws = &h->ws;
    if (!arnoldi_probe(n, k, dbg, *ws, s)) throw InvalidArgument("probe: fused Arnoldi kernel unavailable");
    fn = [=] { arnoldi_probe(n, k, dbg, *ws, s); };
    bytes = 8.0 * n * (2.0 + 2.0 * (k + 1));
    return;
  }
  if (w.rfind("cgs2", 0) == 0) {
    // low-sync Arnoldi step k (lowsync.cu): cgs2.<k> both sweeps,
    // cgs2dots.<k> sweep A, cgs2upd.<k> sweep B. Bytes: each sweep reads
    // V_{0..k-1}, U and w once; sweep B writes v_k and U: 16 n (k+3) per step.
    const int n = h->A.rows;
    const size_t dot = w.find('.');
    const std::string kind = w.substr(0, dot);
    const int k = std::stoi(w.substr(dot + 1));
    const int which = kind == "cgs2dots" ? 1 : kind == "cgs2upd" ? 2 : 3;
    GmresWork* ws = &h->ws;
    if (!lowsync_probe(n, k, *ws, s, which)) throw InvalidArgument("probe: no low-sync step " + w);
    fn = [=] { lowsync_probe(n, k, *ws, s, which); };
    const double sweep = 8.0 * n * (k + 2);
    bytes = (which & 1 ? sweep : 0.0) + (which & 2 ? sweep + 16.0 * n : 0.0);
    return;
  }
  if (w == "precond" || w == "precond.inexact") {
    // one whole MGR application z = M^-1 v through its replayed CUDA graph
    // (the solve's default mode applies dense coarse blocks through their
    // inverses: "precond.inexact"); bytes: the caller's model (solve_model.py)
    MgrHier* HH = &h->H;
    const bool exact = w == "precond";
    fn = [=] { HH->apply_graph(x, y, s, exact); };
    bytes = 0.0;
    return;
  }
  if (w == "spmv.A") {
    const DCsr* A = &h->A;
    fn = [=] { spmv(*A, x, y, s); };
    bytes = spmv_model_bytes(*A);
    return;
  }
  std::string wa = w;
  AmgHier* amg_src = h->H.coarse_amg.get();
  if (w.rfind("mgr.", 0) == 0 && w.find(".frelax.amg.") != std::string::npos) {
    // mgr.<l>.frelax.amg.<k>.<what>: the F-relaxation AMG of MGR level l
    const size_t d = w.find('.', 4);
    const int l = std::stoi(w.substr(4, d - 4));
    if (l < 0 || l >= static_cast<int>(h->H.levels.size())) throw InvalidArgument("probe: no MGR level " + w);
    amg_src = h->H.levels[l].f_relax.amg.get();
    wa = w.substr(w.find(".frelax.") + 8);
  }
  if (wa == w && w.rfind("mgr.", 0) == 0) {
    const size_t d = w.find('.', 4);
    const int l = std::stoi(w.substr(4, d - 4));
    if (l < 0 || l >= static_cast<int>(h->H.levels.size())) throw InvalidArgument("probe: no MGR level " + w);
    MgrLevelD* L = &h->H.levels[l];
    const std::string what = w.substr(d + 1);
    const double nf = static_cast<double>(L->F.size()), nc = static_cast<double>(L->C.size());
    if (what == "rres") {
      if (L->Acf.rows == 0 && nc > 0) throw InvalidArgument("probe: level has no fused restricted residual");
      fn = [=] { spmv_residual(L->Acf, x, y, L->C.get(), z, s); };
      bytes = 12.0 * L->Acf.nnz + 4.0 * (nc + 1) + 8.0 * nf + 16.0 * nc;
      return;
    }
    if (what == "prolong") {
      MgrHier* HH = &h->H;
      fn = [=] { HH->prolong(l, x, y, z, s); };
      bytes = 16.0 * nc + 12.0 * (L->P.nnz - nc) + 4.0 * (nf + 1) + 8.0 * nc + 16.0 * nf;
      return;
    }
  }
  if (wa.rfind("amg.", 0) == 0) {
    const size_t d = wa.find('.', 4);
    const int k = std::stoi(wa.substr(4, d - 4));
    AmgHier* amg = amg_src;
    if (!amg || k < 0 || k + 1 >= static_cast<int>(amg->levels.size())) throw InvalidArgument("probe: no AMG level " + w);
    AmgLevelD* L = &amg->levels[k];
    const std::string what = wa.substr(d + 1);
    const double m = L->A.rows;
    if (what == "resid") {
      fn = [=] { spmv_residual(L->A, x, y, nullptr, z, s); };
      bytes = spmv_model_bytes(L->A) + 8.0 * m;
      return;
    }
    if (what == "pre" || what == "post") {
      BoundRelax* R = what == "pre" ? &L->pre : &L->post;
      fn = [=] { R->apply(y, nullptr, z, s); };
      const double sweep_more = spmv_model_bytes(L->A) + 16.0 * m;  // later sweeps: SpMV + 16m
      bytes = (R->spec.kind == Smoother::jacobi || R->spec.kind == Smoother::l1_jacobi)
                  ? 24.0 * m + (R->spec.sweeps - 1) * sweep_more
                  : R->spec.sweeps * (12.0 * L->A.nnz + 4.0 * (m + 1) + 24.0 * m);
      return;
    }
  }
  throw InvalidArgument("probe: unknown kernel " + w);
}

}  // namespace

extern "C" {

const char* mgrx_last_error(void) { return g_err.c_str(); }

int mgrx_create(const int* devices, int ndev, mgrx_ctx** out) {
  return guarded([&] {
    if (!out) throw InvalidArgument("mgrx_create: null output handle");
    int count = 0;
    MGRX_CK(cudaGetDeviceCount(&count));
    if (count == 0) throw RuntimeError("mgrx_create: no CUDA device visible");
    auto c = std::make_unique<mgrx_ctx>();
    c->device = (devices && ndev > 0) ? devices[0] : 0;
    if (c->device < 0 || c->device >= count) throw InvalidArgument("mgrx_create: device ordinal out of range");
    MGRX_CK(cudaSetDevice(c->device));
    cudaDeviceProp prop;
    MGRX_CK(cudaGetDeviceProperties(&prop, c->device));
    if (prop.major != 10) throw RuntimeError("mgrx_create: libmgrx is built for sm_100a (B200) only");
    MGRX_CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    cudaMemPool_t pool;
    MGRX_CK(cudaDeviceGetDefaultMemPool(&pool, c->device));
    uint64_t thr = UINT64_MAX;
    MGRX_CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    *out = c.release();
    return MGRX_OK;
  });
}

int mgrx_device_memory(mgrx_ctx* ctx, long long* used, long long* reserved, long long* high) {
  return guarded([&] {
    if (!ctx) throw InvalidArgument("mgrx_device_memory: null context");
    use(ctx);
    MGRX_CK(cudaStreamSynchronize(ctx->stream));
    cudaMemPool_t pool;
    MGRX_CK(cudaDeviceGetDefaultMemPool(&pool, ctx->device));
    uint64_t u = 0, r = 0, h = 0;
    MGRX_CK(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &u));
    MGRX_CK(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &r));
    MGRX_CK(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &h));
    if (used) *used = static_cast<long long>(u);
    if (reserved) *reserved = static_cast<long long>(r);
    if (high) *high = static_cast<long long>(h);
    return MGRX_OK;
  });
}

int mgrx_destroy(mgrx_ctx* ctx) {
  return guarded([&] {
    if (ctx) {
      cudaSetDevice(ctx->device);
      cudaStreamSynchronize(ctx->stream);
      cudaStreamDestroy(ctx->stream);
      delete ctx;
    }
    return MGRX_OK;
  });
}

int mgrx_matrix_csr(mgrx_ctx* ctx, int rows, int cols, const int* rowptr, const int* colidx,
                    const double* values, mgrx_mat** out) {
  return guarded([&] {
    use(ctx);
    auto m = std::make_unique<mgrx_mat>();
    m->ctx = ctx;
    m->A = csr_from_host(rows, cols, rowptr, colidx, values, ctx->stream);
    spmv_prepare(m->A, ctx->stream);
    *out = m.release();
    return MGRX_OK;
  });
}

int mgrx_matrix_csr_device(mgrx_ctx* ctx, int rows, int cols, const int* d_rowptr, const int* d_colidx,
                           const double* d_values, mgrx_mat** out) {
  return guarded([&] {
    use(ctx);
    auto m = std::make_unique<mgrx_mat>();
    m->ctx = ctx;
    m->A = csr_from_device(rows, cols, d_rowptr, d_colidx, d_values, ctx->stream);
    spmv_prepare(m->A, ctx->stream);
    *out = m.release();
    return MGRX_OK;
  });
}

int mgrx_matrix_destroy(mgrx_mat* m) {
  return guarded([&] {
    if (m) {
      use(m->ctx);
      MGRX_CK(cudaStreamSynchronize(m->ctx->stream));
      delete m;
    }
    return MGRX_OK;
  });
}

int mgrx_spmv(mgrx_mat* m, const double* x, double* y, int flags) {
  return guarded([&] {
    use(m->ctx);
    cudaStream_t s = m->ctx->stream;
    const bool on_device = (flags & MGRX_ON_DEVICE) != 0;
    TeamSums team_sums((flags & MGRX_TEAM_SUMS) != 0);
    if (on_device) {
      spmv(m->A, x, y, s);
      MGRX_CK(cudaStreamSynchronize(s));
      return MGRX_OK;
    }
    DVec<double> dx(m->A.cols > 0 ? m->A.cols : 1, s), dy(m->A.rows > 0 ? m->A.rows : 1, s);
    dx.upload(x, m->A.cols);
    spmv(m->A, dx.get(), dy.get(), s);
    MGRX_CK(cudaMemcpyAsync(y, dy.get(), sizeof(double) * m->A.rows, cudaMemcpyDeviceToHost, s));
    MGRX_CK(cudaStreamSynchronize(s));
    return MGRX_OK;
  });
}

int mgrx_setup(mgrx_ctx* ctx, mgrx_mat* A, const int* labels, int nfields, const char* const* field_names,
               const int* unknown_map, const char* strategy_json, mgrx_hier** out) {
  return guarded([&] {
    use(ctx);
    if (!A || !labels || !field_names || !strategy_json || !out)
      throw InvalidArgument("mgrx_setup: null argument");
    cudaStream_t s = ctx->stream;
    const Strategy strat = parse_strategy(strategy_json);
    const int n = A->A.rows;
    std::vector<std::string> fields;
    for (int f = 0; f < nfields; ++f) fields.emplace_back(field_names[f]);
    std::vector<int> lab(labels, labels + n);
    for (int v : lab)
      if (v < 0 || v >= nfields) throw InvalidArgument("bundle: label id out of range");
    std::vector<int> umap;
    if (unknown_map) umap.assign(unknown_map, unknown_map + n);
    auto h = std::make_unique<mgrx_hier>();
    h->ctx = ctx;
    const long long b0 = thread_device_bytes();
    EventTimer t(s);
    h->A = csr_copy(A->A, s);
    h->H.setup(h->A, lab, fields, unknown_map ? &umap : nullptr, strat, s);
    spmv_prepare(h->A, s);
    h->H.tune_spmv(s);
    h->setup_s = t.stop();
    h->vin.alloc(n > 0 ? n : 1, s);
    h->vout.alloc(n > 0 ? n : 1, s);
    h->bytes = thread_device_bytes() - b0;
    *out = h.release();
    return MGRX_OK;
  });
}

int mgrx_hier_destroy(mgrx_hier* h) {
  return guarded([&] {
    if (h) {
      use(h->ctx);
      MGRX_CK(cudaStreamSynchronize(h->ctx->stream));
      delete h;
    }
    return MGRX_OK;
  });
}

int mgrx_apply(mgrx_hier* h, const double* v, double* z, int on_device) {
  return guarded([&] {
    use(h->ctx);
    cudaStream_t s = h->ctx->stream;
    const int n = h->A.rows;
    if (on_device) {
      h->H.apply_graph(v, z, s);
    } else {
      h->vin.upload(v, n);
      h->H.apply_graph(h->vin.get(), h->vout.get(), s);
      MGRX_CK(cudaMemcpyAsync(z, h->vout.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    }
    MGRX_CK(cudaStreamSynchronize(s));
    h->H.check(s);
    return MGRX_OK;
  });
}

// gmres(op, b, x, cfg, mgr_preconditioner(h->H)): op is the hierarchy's own
// copy of A (mgrx_solve) or a caller's operator of the same size
// (mgrx_solve_op: the hierarchy kept across Newton steps as a lagged
// preconditioner).
static int solve_with(mgrx_hier* h, const DCsr& op, const double* b, double* x, const mgrx_krylov* cfg,
                      mgrx_report* rep, int flags) {
  const bool on_device = flags & MGRX_ON_DEVICE;
  const bool zero_guess = flags & MGRX_ZERO_GUESS;
  const bool external = &op != &h->A;
  {
    if (!cfg) throw InvalidArgument("mgrx_solve: null config");
    cudaStream_t s = h->ctx->stream;
    const int n = h->A.rows;
    KrylovSpec k;
    k.restart = cfg->restart;
    k.max_iters = cfg->max_iters;
    k.rel_tol = cfg->rel_tol;
    k.abs_tol = cfg->abs_tol;
    k.ortho = cfg->ortho;
    if (k.ortho < 0 || k.ortho > 2) throw InvalidArgument("gmres: unknown orthogonalisation");
    const long long l0 = g_launches;
    const double* db = b;
    double* dx = x;
    if (!on_device) {
      h->vin.upload(b, n);
      if (zero_guess) MGRX_CK(cudaMemsetAsync(h->vout.get(), 0, sizeof(double) * n, s));
      else MGRX_CK(cudaMemcpyAsync(h->vout.get(), x, sizeof(double) * n, cudaMemcpyHostToDevice, s));
      db = h->vin.get();
      dx = h->vout.get();
    } else if (zero_guess) {
      MGRX_CK(cudaMemsetAsync(dx, 0, sizeof(double) * n, s));
    }
    MgrHier* H = &h->H;
    // the bitwise parity mode (MGS) keeps the exact dense substitutions; the
    // default low-sync solve applies dense coarse blocks via their inverses
    const bool exact = k.ortho == kOrthoMgs;
    const DevOp prec = [H, exact](const double* in, double* out, cudaStream_t st) {
      H->apply_graph(in, out, st, exact);
    };
    const DevOp prec_rec = [H, exact](const double* in, double* out, cudaStream_t st) {
      H->apply(in, out, st, exact);
    };
    EventTimer t(s);
    GmresResult r = gmres_device(op, db, dx, k, prec, h->ws, s, prec_rec);
    const double solve_s = t.stop();
    h->H.check(s);
    // the recorded restart cycle is keyed by the operator's address: a
    // caller's matrix may be destroyed and another created in its place
    if (external) h->ws.ls.exec_key = LsWork::Key();
    if (!on_device) {
      MGRX_CK(cudaMemcpyAsync(x, dx, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
      MGRX_CK(cudaStreamSynchronize(s));
    }
    if (rep) {
      rep->converged = r.converged ? 1 : 0;
      rep->iterations = r.iterations;
      rep->final_residual = r.final_residual;
      rep->history_len = static_cast<int>(r.history.size());
      if (rep->history)
        for (int i = 0; i < rep->history_len && i < rep->history_cap; ++i) rep->history[i] = r.history[i];
      rep->setup_s = h->setup_s;
      rep->solve_s = solve_s;
      rep->gpu_launches = g_launches - l0;
    }
    return r.converged ? MGRX_OK : MGRX_NOT_CONVERGED;
  }
}

int mgrx_solve(mgrx_hier* h, const double* b, double* x, const mgrx_krylov* cfg, mgrx_report* rep,
               int flags) {
  return guarded([&] {
    if (!h) throw InvalidArgument("mgrx_solve: null hierarchy");
    use(h->ctx);
    return solve_with(h, h->A, b, x, cfg, rep, flags);
  });
}

int mgrx_solve_op(mgrx_hier* h, mgrx_mat* A, const double* b, double* x, const mgrx_krylov* cfg,
                  mgrx_report* rep, int flags) {
  return guarded([&] {
    if (!h || !A) throw InvalidArgument("mgrx_solve_op: null argument");
    if (A->ctx != h->ctx) throw InvalidArgument("mgrx_solve_op: matrix and hierarchy belong to different contexts");
    if (A->A.rows != A->A.cols) throw InvalidArgument("gmres: matrix must be square");
    if (A->A.rows != h->A.rows) throw InvalidArgument("mgr_apply: size mismatch");
    use(h->ctx);
    return solve_with(h, A->A, b, x, cfg, rep, flags);
  });
}

int mgrx_info(mgrx_hier* h, int* mgr_levels, int* coarse_amg_levels, int* frelax_amg_levels,
              int max_levels) {
  return guarded([&] {
    *mgr_levels = static_cast<int>(h->H.levels.size());
    *coarse_amg_levels = h->H.coarse_amg ? static_cast<int>(h->H.coarse_amg->levels.size()) : 0;
    for (int l = 0; l < *mgr_levels && l < max_levels; ++l) {
      const auto& amg = h->H.levels[l].f_relax.amg;
      frelax_amg_levels[l] = amg ? static_cast<int>(amg->levels.size()) : 0;
    }
    return MGRX_OK;
  });
}

int mgrx_amg_info(mgrx_hier* h, int which, int* nlevels, int* level_sizes, int cap, long long* fallback_rows,
                  int* truncated) {
  return guarded([&] {
    const AmgHier* amg = nullptr;
    if (which < 0) amg = h->H.coarse_amg.get();
    else if (which < static_cast<int>(h->H.levels.size())) amg = h->H.levels[which].f_relax.amg.get();
    if (!amg) throw InvalidArgument("mgrx_amg_info: no AMG hierarchy at " + std::to_string(which));
    *nlevels = static_cast<int>(amg->level_sizes.size());
    for (int i = 0; i < *nlevels && i < cap; ++i) level_sizes[i] = amg->level_sizes[i];
    *fallback_rows = amg->fallback_rows;
    *truncated = amg->truncated ? 1 : 0;
    return MGRX_OK;
  });
}

int mgrx_corrupt_transfer(mgrx_hier* h, int level, double factor) {
  return guarded([&] {
    use(h->ctx);
    h->H.corrupt_transfer(level, factor, h->ctx->stream);
    // the recorded restart cycle embeds the clean preconditioner
    if (h->ws.ls.exec) cudaGraphExecDestroy(h->ws.ls.exec);
    h->ws.ls.exec = nullptr;
    h->ws.ls.exec_key = {};
    return MGRX_OK;
  });
}

int mgrx_dump(mgrx_hier* h, const char* path_c, int* kind, int* rows, int* cols, long long* nnz, int* ptr,
              int* col, double* val) {
  return guarded([&] {
    use(h->ctx);
    cudaStream_t s = h->ctx->stream;
    const std::string path(path_c);
    const DCsr* csr = nullptr;
    const DVec<int>* ints = nullptr;
    const std::vector<int>* hints = nullptr;
    const DVec<double>* vec = nullptr;
    auto amg_fields = [&](AmgHier* amg, const std::string& rest) {
      const size_t d = rest.find('.');
      const int kk = std::stoi(rest.substr(0, d));
      const std::string what = rest.substr(d + 1);
      if (!amg || kk < 0 || kk >= static_cast<int>(amg->levels.size()))
        throw InvalidArgument("dump: no AMG level " + path);
      AmgLevelD& L = amg->levels[kk];
      if (what == "A") csr = &L.A;
      else if (what == "P") csr = &L.P;
      else if (what == "R") csr = &L.R;
      else if (what == "C") ints = &L.C;
      else if (what == "F") ints = &L.F;
      else if (what == "l1d") vec = &L.pre.l1d;
      else if (what == "dinv") vec = &L.pre.dinv;
      else if (what == "umap") hints = &L.umap;
    };
    if (path.rfind("mgr.coarse.amg.", 0) == 0) {
      amg_fields(h->H.coarse_amg.get(), path.substr(15));
    } else if (path == "mgr.coarse.A") {
      csr = &h->H.A_coarse;
    } else if (path.rfind("mgr.", 0) == 0) {
      const size_t d = path.find('.', 4);
      const int l = std::stoi(path.substr(4, d - 4));
      if (l < 0 || l >= static_cast<int>(h->H.levels.size())) throw InvalidArgument("dump: no MGR level " + path);
      MgrLevelD& L = h->H.levels[l];
      const std::string what = path.substr(d + 1);
      if (what.rfind("frelax.amg.", 0) == 0) amg_fields(L.f_relax.amg.get(), what.substr(11));
      else if (what == "A") csr = &L.A;
      else if (what == "P") csr = &L.P;
      else if (what == "R") csr = &L.R;
      else if (what == "F") ints = &L.F;
      else if (what == "C") ints = &L.C;
      else if (what == "frelax.dinv") vec = &L.f_relax.dinv;
    }
    if (csr) {
      *kind = 0;
      *rows = csr->rows;
      *cols = csr->cols;
      *nnz = csr->nnz;
      if (ptr) MGRX_CK(cudaMemcpyAsync(ptr, csr->ptr.get(), sizeof(int) * (csr->rows + 1), cudaMemcpyDeviceToHost, s));
      if (col && csr->nnz) MGRX_CK(cudaMemcpyAsync(col, csr->col.get(), sizeof(int) * csr->nnz, cudaMemcpyDeviceToHost, s));
      if (val && csr->nnz) MGRX_CK(cudaMemcpyAsync(val, csr->val.get(), sizeof(double) * csr->nnz, cudaMemcpyDeviceToHost, s));
      MGRX_CK(cudaStreamSynchronize(s));
      return MGRX_OK;
    }
    if (ints) {
      *kind = 1;
      *rows = static_cast<int>(ints->size());
      *cols = 1;
      *nnz = static_cast<long long>(ints->size());
      if (col && ints->size()) MGRX_CK(cudaMemcpyAsync(col, ints->get(), sizeof(int) * ints->size(), cudaMemcpyDeviceToHost, s));
      MGRX_CK(cudaStreamSynchronize(s));
      return MGRX_OK;
    }
    if (hints) {
      *kind = 1;
      *rows = static_cast<int>(hints->size());
      *cols = 1;
      *nnz = static_cast<long long>(hints->size());
      if (col && !hints->empty()) std::memcpy(col, hints->data(), sizeof(int) * hints->size());
      return MGRX_OK;
    }
    if (vec) {
      *kind = 2;
      *rows = static_cast<int>(vec->size());
      *cols = 1;
      *nnz = static_cast<long long>(vec->size());
      if (val && vec->size()) MGRX_CK(cudaMemcpyAsync(val, vec->get(), sizeof(double) * vec->size(), cudaMemcpyDeviceToHost, s));
      MGRX_CK(cudaStreamSynchronize(s));
      return MGRX_OK;
    }
    throw InvalidArgument("dump: unknown path " + path);
  });
}

int mgrx_time_kernel(mgrx_hier* h, const char* which, int reps, double* avg_ms, double* bytes) {
  return guarded([&] {
    use(h->ctx);
    cudaStream_t s = h->ctx->stream;
    std::function<void()> fn;
    double b = 0.0;
    std::string w(which);
    // "cold:<probe>": the launch's duration from a cold L2, measured without
    // launch latency as the difference of two back-to-back streams of `reps`
    // iterations, [256 MB flush read, launch] and [flush read] alone
    const bool cold = w.rfind("cold:", 0) == 0;
    if (cold) w = w.substr(5);
    prepare_probe(h, w, fn, b, s);
    // probes time the kernels of the default (tolerance-level) solve;
    // MGRX_PROBE_EXACT=1: the bitwise kernels
    static const bool probe_exact = [] {
      const char* e = std::getenv("MGRX_PROBE_EXACT");
      return e && e[0] == '1';
    }();
    TeamSums team_sums(!probe_exact);
    for (int i = 0; i < 3; ++i) fn();  // warm-up
    // Default: launches back to back (the L2 keeps whatever of the previous
    // launch's inputs fits in 126 MB: kernels whose working set is near the L2
    // size read part of it from L2). MGRX_PROBE_FLUSH=1: each timed launch
    // starts from a cold L2 (256 MB read before it, outside its event
    // pair; the per-launch events then include ~5 us of launch latency).
    static const bool flush = [] {
      const char* e = std::getenv("MGRX_PROBE_FLUSH");
      return e && e[0] == '1';
    }();
    if (cold) {
      constexpr size_t kFlush = 256ull << 20;
      if (h->flushbuf.size() < kFlush) {
        h->flushbuf.alloc(kFlush, s);
        h->flushbuf.zero();
      }
      const int n = reps > 0 ? reps : 1;
      double best_with = 1e300, best_without = 1e300;
      for (int round = 0; round < 3; ++round) {
        for (int i = 0; i < 2; ++i) l2_flush_read(h->flushbuf.get(), kFlush, s);
        {
          EventTimer t(s);
          for (int i = 0; i < n; ++i) l2_flush_read(h->flushbuf.get(), kFlush, s);
          best_without = std::min(best_without, t.stop());
        }
        {
          EventTimer t(s);
          for (int i = 0; i < n; ++i) {
            l2_flush_read(h->flushbuf.get(), kFlush, s);
            fn();
          }
          best_with = std::min(best_with, t.stop());
        }
      }
      *avg_ms = (best_with - best_without) * 1e3 / n;
    } else if (!flush) {
      EventTimer t(s);
      for (int i = 0; i < reps; ++i) fn();
      *avg_ms = t.stop() * 1e3 / (reps > 0 ? reps : 1);
    } else {
      constexpr size_t kFlush = 256ull << 20;
      if (h->flushbuf.size() < kFlush) {
        h->flushbuf.alloc(kFlush, s);
        h->flushbuf.zero();
      }
      cudaEvent_t e0, e1;
      MGRX_CK(cudaEventCreate(&e0));
      MGRX_CK(cudaEventCreate(&e1));
      double tot = 0.0;
      for (int i = 0; i < reps; ++i) {
        l2_flush_read(h->flushbuf.get(), kFlush, s);
        MGRX_CK(cudaEventRecord(e0, s));
        fn();
        MGRX_CK(cudaEventRecord(e1, s));
        MGRX_CK(cudaEventSynchronize(e1));
        float ms = 0.f;
        MGRX_CK(cudaEventElapsedTime(&ms, e0, e1));
        tot += ms;
      }
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      *avg_ms = tot / (reps > 0 ? reps : 1);
    }
    *bytes = b;
    return MGRX_OK;
  });
}

// ---------------------------------------------------------------------------
// Row-slab sharded solve
// ---------------------------------------------------------------------------
int mgrx_nccl_unique_id(unsigned char* out) {
  return guarded([&] {
    if (!out) throw InvalidArgument("mgrx_nccl_unique_id: null buffer");
    nccl_unique_id(out);
    return MGRX_OK;
  });
}

int mgrx_local_group_create(int size, mgrx_group** out) {
  return guarded([&] {
    if (size < 1 || !out) throw InvalidArgument("mgrx_local_group_create: bad arguments");
    auto* g = new mgrx_group;
    g->hub = make_local_hub(size);
    g->size = size;
    *out = g;
    return MGRX_OK;
  });
}

int mgrx_transport_group_create(int size, const mgrx_transport* t, mgrx_group** out) {
  return guarded([&] {
    if (size < 1 || !out || !t || !t->exchange || !t->allgather)
      throw InvalidArgument("mgrx_transport_group_create: size >= 1 and both transport functions are required");
    auto* g = new mgrx_group;
    g->size = size;
    g->host = true;
    g->tr.user = t->user;
    g->tr.exchange = t->exchange;
    g->tr.allgather = t->allgather;
    *out = g;
    return MGRX_OK;
  });
}

int mgrx_local_group_destroy(mgrx_group* g) {
  delete g;
  return MGRX_OK;
}

int mgrx_shard_create(mgrx_hier* h, int rank, int size, const int* row_starts, const unsigned char* nccl_id,
                      mgrx_group* group, mgrx_shard** out) {
  return guarded([&] {
    use(h->ctx);
    if (!out || size < 1 || rank < 0 || rank >= size) throw InvalidArgument("mgrx_shard_create: bad rank/size");
    if ((nccl_id == nullptr) == (group == nullptr) && size > 1)
      throw InvalidArgument("mgrx_shard_create: give exactly one of nccl_id and group");
    const int n = h->A.rows;
    std::vector<int> st(size + 1);
    if (row_starts) {
      st.assign(row_starts, row_starts + size + 1);
    } else {
      for (int q = 0; q <= size; ++q) st[q] = static_cast<int>(static_cast<long long>(n) * q / size);
    }
    std::unique_ptr<Comm> cm;
    if (group) {
      if (group->size != size) throw InvalidArgument("mgrx_shard_create: group size mismatch");
      cm = group->comm(rank);
    } else if (nccl_id) {
      cm = make_nccl_comm(nccl_id, rank, size);
    } else {
      auto hub = make_local_hub(1);
      cm = make_local_comm(hub, 0);
    }
    auto* sd = new mgrx_shard;
    sd->ctx = h->ctx;
    sd->setup_s = h->setup_s;
    const long long b0 = thread_device_bytes();
    try {
      MGRX_CK(cudaStreamCreateWithFlags(&sd->stream, cudaStreamNonBlocking));
      MGRX_CK(cudaStreamSynchronize(h->ctx->stream));
      sd->sh = std::make_unique<Shard>();
      sd->sh->build(h->H, h->A, st, std::move(cm), sd->stream);
      const int own = sd->sh->row_end - sd->sh->row_begin;
      sd->vin.alloc(own, sd->stream);
      sd->vout.alloc(own, sd->stream);
      sd->bytes = thread_device_bytes() - b0;
    } catch (...) {
      delete sd;
      throw;
    }
    *out = sd;
    return MGRX_OK;
  });
}

int mgrx_shard_create_scatter(mgrx_ctx* ctx, mgrx_hier* h, int rank, int size, const int* row_starts,
                              const unsigned char* nccl_id, mgrx_group* group, mgrx_shard** out) {
  return guarded([&] {
    if (!ctx || !out || size < 1 || rank < 0 || rank >= size)
      throw InvalidArgument("mgrx_shard_create_scatter: bad rank/size");
    use(ctx);
    if ((rank == 0) != (h != nullptr))
      throw InvalidArgument("mgrx_shard_create_scatter: rank 0 (and only rank 0) passes the global hierarchy");
    if (!row_starts) throw InvalidArgument("mgrx_shard_create_scatter: row starts are required");
    if ((nccl_id == nullptr) == (group == nullptr) && size > 1)
      throw InvalidArgument("mgrx_shard_create_scatter: give exactly one of nccl_id and group");
    const std::vector<int> st(row_starts, row_starts + size + 1);
    std::unique_ptr<Comm> cm;
    if (group) {
      if (group->size != size) throw InvalidArgument("mgrx_shard_create_scatter: group size mismatch");
      cm = group->comm(rank);
    } else if (nccl_id) {
      cm = make_nccl_comm(nccl_id, rank, size);
    } else {
      auto hub = make_local_hub(1);
      cm = make_local_comm(hub, 0);
    }
    auto* sd = new mgrx_shard;
    sd->ctx = ctx;
    const long long b0 = thread_device_bytes();
    try {
      const auto t0 = std::chrono::steady_clock::now();
      MGRX_CK(cudaStreamCreateWithFlags(&sd->stream, cudaStreamNonBlocking));
      MGRX_CK(cudaStreamSynchronize(ctx->stream));
      sd->sh = std::make_unique<Shard>();
      sd->sh->build_scatter(h ? &h->H : nullptr, h ? &h->A : nullptr, st, std::move(cm), sd->stream);
      const int own = sd->sh->row_end - sd->sh->row_begin;
      sd->vin.alloc(own, sd->stream);
      sd->vout.alloc(own, sd->stream);
      MGRX_CK(cudaStreamSynchronize(sd->stream));
      sd->setup_s = (h ? h->setup_s : 0.0) +
                    std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      sd->bytes = thread_device_bytes() - b0;
    } catch (...) {
      delete sd;
      throw;
    }
    *out = sd;
    return MGRX_OK;
  });
}

int mgrx_hier_bytes(mgrx_hier* h, long long* bytes) {
  return guarded([&] {
    if (!h || !bytes) throw InvalidArgument("mgrx_hier_bytes: null argument");
    *bytes = h->bytes;
    return MGRX_OK;
  });
}

int mgrx_shard_bytes(mgrx_shard* sd, long long* bytes) {
  return guarded([&] {
    if (!sd || !bytes) throw InvalidArgument("mgrx_shard_bytes: null argument");
    *bytes = sd->bytes;
    return MGRX_OK;
  });
}

int mgrx_shard_rows(mgrx_shard* sd, int* row_begin, int* row_end) {
  return guarded([&] {
    *row_begin = sd->sh->row_begin;
    *row_end = sd->sh->row_end;
    return MGRX_OK;
  });
}

int mgrx_shard_fused(mgrx_shard* sd, int* fused) {
  return guarded([&] {
    if (!fused) throw InvalidArgument("mgrx_shard_fused: null output");
    *fused = sd->sh->fused ? 1 : 0;
    return MGRX_OK;
  });
}

int mgrx_shard_apply(mgrx_shard* sd, const double* v, double* z, int on_device) {
  return guarded([&] {
    use(sd->ctx);
    const int n = sd->sh->row_end - sd->sh->row_begin;
    cudaStream_t s = sd->stream;
    if (on_device) {
      sd->sh->apply(v, z);
      return MGRX_OK;
    }
    sd->vin.upload(v, n);
    sd->sh->apply(sd->vin.get(), sd->vout.get());
    MGRX_CK(cudaMemcpyAsync(z, sd->vout.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    MGRX_CK(cudaStreamSynchronize(s));
    return MGRX_OK;
  });
}

int mgrx_shard_solve(mgrx_shard* sd, const double* b, double* x, const mgrx_krylov* cfg, mgrx_report* rep,
                     int flags) {
  const bool on_device = flags & MGRX_ON_DEVICE;
  const bool zero_guess = flags & MGRX_ZERO_GUESS;
  return guarded([&] {
    use(sd->ctx);
    if (!cfg) throw InvalidArgument("mgrx_shard_solve: null config");
    cudaStream_t s = sd->stream;
    const int n = sd->sh->row_end - sd->sh->row_begin;
    KrylovSpec k;
    k.restart = cfg->restart;
    k.max_iters = cfg->max_iters;
    k.rel_tol = cfg->rel_tol;
    k.abs_tol = cfg->abs_tol;
    k.ortho = cfg->ortho;
    if (k.ortho < 0 || k.ortho > 2) throw InvalidArgument("gmres: unknown orthogonalisation");
    const long long l0 = g_launches;
    const double* db = b;
    double* dx = x;
    if (!on_device) {
      sd->vin.upload(b, n);
      if (zero_guess) MGRX_CK(cudaMemsetAsync(sd->vout.get(), 0, sizeof(double) * n, s));
      else MGRX_CK(cudaMemcpyAsync(sd->vout.get(), x, sizeof(double) * n, cudaMemcpyHostToDevice, s));
      db = sd->vin.get();
      dx = sd->vout.get();
    } else if (zero_guess) {
      MGRX_CK(cudaMemsetAsync(dx, 0, sizeof(double) * n, s));
    }
    EventTimer t(s);
    GmresResult r = sd->sh->solve(db, dx, k);
    const double solve_s = t.stop();
    if (!on_device) {
      MGRX_CK(cudaMemcpyAsync(x, dx, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
      MGRX_CK(cudaStreamSynchronize(s));
    }
    if (rep) {
      rep->converged = r.converged ? 1 : 0;
      rep->iterations = r.iterations;
      rep->final_residual = r.final_residual;
      rep->history_len = static_cast<int>(r.history.size());
      if (rep->history)
        for (int i = 0; i < rep->history_len && i < rep->history_cap; ++i) rep->history[i] = r.history[i];
      rep->setup_s = sd->setup_s;
      rep->solve_s = solve_s;
      rep->gpu_launches = g_launches - l0;
    }
    return r.converged ? MGRX_OK : MGRX_NOT_CONVERGED;
  });
}

int mgrx_shard_destroy(mgrx_shard* sd) {
  return guarded([&] {
    if (sd) use(sd->ctx);
    delete sd;
    return MGRX_OK;
  });
}

}  // extern "C"
