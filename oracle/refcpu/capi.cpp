// refcpu — CPU ORACLE (test infrastructure only; see csr.hpp header).
// Plain C entry points so tests/ and bench.py can drive the oracle through
// ctypes. Status codes mirror proj/tools/mgr_main.cpp:34 (0 ok, 1 not
// converged, 2 invalid argument, 3 runtime error).
#include <chrono>
#include <cstring>
#include <memory>
#include <string>

#include "solver.hpp"

using namespace refcpu;

namespace {

thread_local std::string g_err;

int fail_code(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const std::invalid_argument*>(&e)) return 2;
  return 3;
}

struct RefHandle {
  Csr A;
  MgrHierarchy H;
  double setup_s = 0;
};

Csr make_csr(int n, int ncols, const int* ptr, const int* col, const double* val) {
  Csr A;
  A.rows = n;
  A.cols = ncols;
  A.ptr.assign(ptr, ptr + n + 1);
  A.col.assign(col, col + ptr[n]);
  A.val.assign(val, val + ptr[n]);
  validate(A);
  return A;
}

// Path grammar shared with libmgrx's mgrx_dump:
//   mgr.<l>.{A,P,R,F,C,frelax.dinv}   mgr.coarse.A
//   mgr.<l>.frelax.amg.<k>.{A,P,R,C,F}   mgr.coarse.amg.<k>.{A,P,R,C,F}
const AmgHierarchy* amg_at(const RefHandle& h, const std::string& pfx, size_t& off) {
  if (pfx.rfind("mgr.coarse.amg.", 0) == 0) {
    off = std::strlen("mgr.coarse.amg.");
    return h.H.coarse_amg.get();
  }
  if (pfx.rfind("mgr.", 0) == 0) {
    const size_t d = pfx.find('.', 4);
    if (d == std::string::npos) return nullptr;
    const std::string lvl = pfx.substr(4, d - 4);
    if (lvl == "coarse") return nullptr;
    const int l = std::stoi(lvl);
    const std::string rest = pfx.substr(d + 1);
    if (rest.rfind("frelax.amg.", 0) == 0 && l < h.H.num_reduction_levels()) {
      off = d + 1 + std::strlen("frelax.amg.");
      return h.H.levels[l].f_relax.amg_hierarchy();
    }
  }
  return nullptr;
}

struct DumpTarget {
  const Csr* csr = nullptr;
  const IndexList* ints = nullptr;
  const std::vector<int>* ints2 = nullptr;
  const Vec* vec = nullptr;
};

DumpTarget resolve(const RefHandle& h, const std::string& path) {
  DumpTarget t;
  size_t off = 0;
  if (const AmgHierarchy* amg = amg_at(h, path, off)) {
    const size_t d = path.find('.', off);
    const int k = std::stoi(path.substr(off, d - off));
    const std::string what = path.substr(d + 1);
    if (k < 0 || k >= amg->num_levels()) throw std::invalid_argument("dump: no AMG level " + path);
    const AmgLevel& L = amg->levels[k];
    if (what == "A") t.csr = &L.A;
    else if (what == "P") t.csr = &L.P;
    else if (what == "R") t.csr = &L.R;
    else if (what == "C") t.ints = &L.C;
    else if (what == "F") t.ints = &L.F;
    else if (what == "l1d") t.vec = &L.pre.l1d();
    else if (what == "dinv") t.vec = &L.pre.dinv();
    else if (what == "umap") t.ints2 = &L.unknown_map;
    return t;
  }
  if (path == "mgr.coarse.A") {
    t.csr = &h.H.A_coarse;
    return t;
  }
  if (path.rfind("mgr.", 0) == 0) {
    const size_t d = path.find('.', 4);
    const int l = std::stoi(path.substr(4, d - 4));
    if (l < 0 || l >= h.H.num_reduction_levels()) throw std::invalid_argument("dump: no MGR level " + path);
    const MgrLevel& L = h.H.levels[l];
    const std::string what = path.substr(d + 1);
    if (what == "A") t.csr = &L.A;
    else if (what == "P") t.csr = &L.P;
    else if (what == "R") t.csr = &L.R;
    else if (what == "F") t.ints = &L.F;
    else if (what == "C") t.ints = &L.C;
    else if (what == "frelax.dinv") t.vec = &L.f_relax.dinv();
  }
  return t;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_set_threads(int n) { set_threads(n); }
void ref_set_dot_order(int m) { set_dot_order(m); }

int ref_spmv(int n, int ncols, const int* ptr, const int* col, const double* val, const double* x,
             double* y) {
  try {
    const Csr A = make_csr(n, ncols, ptr, col, val);
    const Vec xv(x, x + ncols);
    const Vec yv = spmv(A, xv);
    std::memcpy(y, yv.data(), sizeof(double) * n);
    return 0;
  } catch (const std::exception& e) {
    return fail_code(e);
  }
}

int ref_setup(int n, const int* ptr, const int* col, const double* val, const int* labels,
              int nfields, const char* const* field_names, const int* unknown_map,
              const char* strategy_json, void** out) {
  try {
    auto h = std::make_unique<RefHandle>();
    h->A = make_csr(n, n, ptr, col, val);
    DofPartition part;
    for (int f = 0; f < nfields; ++f) part.field_order.emplace_back(field_names[f]);
    part.labels.assign(labels, labels + n);
    for (int i = 0; i < n; ++i)
      if (labels[i] < 0 || labels[i] >= nfields) throw std::invalid_argument("label id out of range");
    const MgrStrategy s = strategy_from_json_text(strategy_json);
    std::vector<int> umap;
    if (unknown_map) umap.assign(unknown_map, unknown_map + n);
    const auto t0 = std::chrono::steady_clock::now();
    h->H = mgr_setup(h->A, part, s, unknown_map ? &umap : nullptr);
    h->setup_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = h.release();
    return 0;
  } catch (const std::exception& e) {
    return fail_code(e);
  }
}

double ref_setup_seconds(void* hp) { return static_cast<RefHandle*>(hp)->setup_s; }

int ref_apply(void* hp, const double* v, double* z) {
  try {
    auto* h = static_cast<RefHandle*>(hp);
    const Vec vv(v, v + h->A.rows);
    const Vec zz = mgr_apply(h->H, vv);
    std::memcpy(z, zz.data(), sizeof(double) * zz.size());
    return 0;
  } catch (const std::exception& e) {
    return fail_code(e);
  }
}

// report: converged, iterations, history_len written; history has history_cap slots.
int ref_solve(void* hp, const double* b, double* x, int restart, int max_iters, double rel_tol,
              double abs_tol, int* converged, int* iterations, double* final_residual,
              double* history, int history_cap, int* history_len, double* solve_s) {
  try {
    auto* h = static_cast<RefHandle*>(hp);
    const Index n = h->A.rows;
    KrylovConfig kc;
    kc.restart = restart;
    kc.max_iters = max_iters;
    kc.rel_tol = rel_tol;
    kc.abs_tol = abs_tol;
    const Vec bv(b, b + n);
    Vec xv(x, x + n);
    const auto t0 = std::chrono::steady_clock::now();
    const SolveReport rep = gmres(h->A, bv, xv, kc, mgr_preconditioner(h->H));
    *solve_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::memcpy(x, xv.data(), sizeof(double) * n);
    *converged = rep.converged ? 1 : 0;
    *iterations = rep.iterations;
    *final_residual = rep.final_residual;
    const int len = static_cast<int>(rep.residual_history.size());
    *history_len = len;
    for (int i = 0; i < len && i < history_cap; ++i) history[i] = rep.residual_history[i];
    return rep.converged ? 0 : 1;
  } catch (const std::exception& e) {
    return fail_code(e);
  }
}

// gmres(A', b, x, cfg, mgr_preconditioner(H)) with an operator A' other than
// the one H was built from (proj/include/mgrkit/krylov.hpp:33-34 takes the
// operator and the preconditioner separately).
int ref_solve_op(void* hp, int n, const int* ptr, const int* col, const double* val, const double* b,
                 double* x, int restart, int max_iters, double rel_tol, double abs_tol, int* converged,
                 int* iterations, double* final_residual, double* history, int history_cap,
                 int* history_len) {
  try {
    auto* h = static_cast<RefHandle*>(hp);
    const Csr A = make_csr(n, n, ptr, col, val);
    KrylovConfig kc;
    kc.restart = restart;
    kc.max_iters = max_iters;
    kc.rel_tol = rel_tol;
    kc.abs_tol = abs_tol;
    const Vec bv(b, b + n);
    Vec xv(x, x + n);
    const SolveReport rep = gmres(A, bv, xv, kc, mgr_preconditioner(h->H));
    std::memcpy(x, xv.data(), sizeof(double) * n);
    *converged = rep.converged ? 1 : 0;
    *iterations = rep.iterations;
    *final_residual = rep.final_residual;
    const int len = static_cast<int>(rep.residual_history.size());
    *history_len = len;
    for (int i = 0; i < len && i < history_cap; ++i) history[i] = rep.residual_history[i];
    return rep.converged ? 0 : 1;
  } catch (const std::exception& e) {
    return fail_code(e);
  }
}

// Two-call protocol: pass null buffers to query sizes. kind: 0 csr, 1 int list, 2 vector.
int ref_dump(void* hp, const char* path, int* kind, int* rows, int* cols, long long* nnz, int* ptr,
             int* col, double* val) {
  try {
    auto* h = static_cast<RefHandle*>(hp);
    const DumpTarget t = resolve(*h, path);
    if (t.csr) {
      *kind = 0;
      *rows = t.csr->rows;
      *cols = t.csr->cols;
      *nnz = t.csr->nnz();
      if (ptr) std::memcpy(ptr, t.csr->ptr.data(), sizeof(int) * (t.csr->rows + 1));
      if (col) std::memcpy(col, t.csr->col.data(), sizeof(int) * t.csr->nnz());
      if (val) std::memcpy(val, t.csr->val.data(), sizeof(double) * t.csr->nnz());
      return 0;
    }
    const std::vector<int>* iv = t.ints ? t.ints : t.ints2;
    if (iv) {
      *kind = 1;
      *rows = static_cast<int>(iv->size());
      *cols = 1;
      *nnz = static_cast<long long>(iv->size());
      if (col) std::memcpy(col, iv->data(), sizeof(int) * iv->size());
      return 0;
    }
    if (t.vec) {
      *kind = 2;
      *rows = static_cast<int>(t.vec->size());
      *cols = 1;
      *nnz = static_cast<long long>(t.vec->size());
      if (val) std::memcpy(val, t.vec->data(), sizeof(double) * t.vec->size());
      return 0;
    }
    throw std::invalid_argument(std::string("dump: unknown path ") + path);
  } catch (const std::exception& e) {
    return fail_code(e);
  }
}

// Hierarchy shape: number of MGR levels and AMG levels (coarse / per F-relax).
int ref_info(void* hp, int* mgr_levels, int* coarse_amg_levels, int* frelax_amg_levels,
             int max_levels) {
  auto* h = static_cast<RefHandle*>(hp);
  *mgr_levels = h->H.num_reduction_levels();
  *coarse_amg_levels = h->H.coarse_amg ? h->H.coarse_amg->num_levels() : 0;
  for (int l = 0; l < h->H.num_reduction_levels() && l < max_levels; ++l) {
    const AmgHierarchy* a = h->H.levels[l].f_relax.amg_hierarchy();
    frelax_amg_levels[l] = a ? a->num_levels() : 0;
  }
  return 0;
}

int ref_amg_info(void* hp, int which, int* nlevels, int* level_sizes, int cap, long long* fallback_rows,
                 int* truncated) {
  auto* h = static_cast<RefHandle*>(hp);
  const AmgHierarchy* a = nullptr;
  if (which < 0) a = h->H.coarse_amg ? h->H.coarse_amg.get() : nullptr;
  else if (which < h->H.num_reduction_levels()) a = h->H.levels[which].f_relax.amg_hierarchy();
  if (!a) {
    g_err = "no AMG hierarchy";
    return 2;
  }
  *nlevels = static_cast<int>(a->info.level_sizes.size());
  for (int i = 0; i < *nlevels && i < cap; ++i) level_sizes[i] = a->info.level_sizes[i];
  *fallback_rows = a->info.interp_fallback_rows;
  *truncated = a->info.truncated ? 1 : 0;
  return 0;
}

void ref_free(void* hp) { delete static_cast<RefHandle*>(hp); }

}  // extern "C"
