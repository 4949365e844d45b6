// refcpu — CPU ORACLE (test infrastructure only; see csr.hpp header).
// Restates proj/include/mgrkit/{relax,amg,mgr,krylov}.hpp semantics.
#pragma once

#include <functional>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "csr.hpp"

namespace refcpu {

// ---- relax (proj/include/mgrkit/relax.hpp:21-92) ---------------------------
enum class SmootherKind {
  jacobi,
  l1_jacobi,
  hybrid_l1_gs_forward,
  hybrid_l1_gs_backward,
  block_jacobi_exact,
  amg_vcycle,
  dense_lu,
};
using Partition = std::vector<std::pair<Index, Index>>;

struct AmgConfig;
struct AmgHierarchy;

struct SmootherSpec {
  SmootherKind kind = SmootherKind::jacobi;
  Index sweeps = 1;
  Real weight = 1.0;
  std::vector<Index> block_sizes;
  Partition partition;
  std::shared_ptr<const AmgConfig> amg;
  bool use_unknown_map = false;
};

Vec l1_diagonal(const Csr& A, const Partition& partition);            // relax.cpp:34-48
void jacobi_sweep(const Csr& A, const Vec& b, Vec& x, Real weight);   // relax.cpp:50-53
void hybrid_l1_gs_sweep(const Csr& A, const Vec& l1d, const Vec& b, Vec& x, bool forward,
                        const Partition& partition);                  // relax.cpp:55-78
void hybrid_l1_gs_sweep(const Csr& A, const Vec& b, Vec& x, bool forward,
                        const Partition& partition = {});

class BoundSmoother {
 public:
  static BoundSmoother bind(const SmootherSpec& spec, const Csr& A,
                            const std::vector<int>* unknown_map = nullptr);  // relax.cpp:90-149
  Vec apply(const Vec& r) const;                                             // relax.cpp:151-192
  bool bound() const { return static_cast<bool>(A_); }
  const SmootherSpec& spec() const { return spec_; }
  const AmgHierarchy* amg_hierarchy() const { return amg_.get(); }
  const Vec& dinv() const { return dinv_; }
  const Vec& l1d() const { return l1d_; }

 private:
  SmootherSpec spec_;
  std::shared_ptr<const Csr> A_;
  Partition partition_;
  Vec dinv_, l1d_;
  std::shared_ptr<BlockDiagonalLU> block_lu_;
  std::shared_ptr<DenseLU> dense_lu_;
  std::shared_ptr<AmgHierarchy> amg_;
};

// ---- amg (proj/include/mgrkit/amg.hpp:14-71) -------------------------------
struct AmgConfig {
  Real strength_theta = 0.25;
  Index max_levels = 25;
  Index coarse_size = 50;
  SmootherSpec pre_smoother{SmootherKind::hybrid_l1_gs_forward, 1, 1.0, {}, {}, nullptr, false};
  SmootherSpec post_smoother{SmootherKind::hybrid_l1_gs_backward, 1, 1.0, {}, {}, nullptr, false};
  std::vector<int> unknown_map;
};

struct AmgLevel {
  Csr A, P, R;
  BoundSmoother pre, post;
  std::vector<int> unknown_map;
  IndexList C, F;  // splitting that produced P (instrumentation for parity)
};

struct AmgSetupInfo {
  std::vector<Index> level_sizes;
  Index interp_fallback_rows = 0;
  bool truncated = false;
};

struct AmgHierarchy {
  std::vector<AmgLevel> levels;
  DenseLU coarse_solver;
  AmgSetupInfo info;
  Index num_levels() const { return static_cast<Index>(levels.size()); }
  Index fine_size() const { return levels.empty() ? 0 : levels.front().A.rows; }
};

Csr strength_graph(const Csr& A, Real theta);                          // amg.cpp:11-34
void pmis_coarsen(const Csr& S, IndexList& C, IndexList& F);           // amg.cpp:36-86
Csr classical_interp(const Csr& A, const Csr& S, const IndexList& C, const IndexList& F,
                     Index* fallback_rows = nullptr);                  // amg.cpp:88-141
AmgHierarchy amg_setup(const Csr& A, const AmgConfig& cfg);            // amg.cpp:246-291
Vec amg_vcycle(const AmgHierarchy& H, const Vec& r);                   // amg.cpp:293-297

// ---- krylov (proj/include/mgrkit/krylov.hpp:12-38) -------------------------
using LinOp = std::function<Vec(const Vec&)>;
struct KrylovConfig {
  Index restart = 50;
  Index max_iters = 500;
  Real rel_tol = 1e-7;
  Real abs_tol = 0.0;
};
struct SolveReport {
  bool converged = false;
  Index iterations = 0;
  Real final_residual = 0.0;
  std::vector<Real> residual_history;
};
SolveReport gmres(const Csr& A, const Vec& b, Vec& x, const KrylovConfig& cfg,
                  const LinOp& preconditioner = {});                  // krylov.cpp:149-154
SolveReport gmres_op(const LinOp& A, Index n, const Vec& b, Vec& x, const KrylovConfig& cfg,
                     const LinOp& preconditioner = {});               // krylov.cpp:37-147

// ---- mgr (proj/include/mgrkit/mgr.hpp:20-114) ------------------------------
struct DofPartition {
  std::vector<std::string> field_order;
  std::vector<Index> labels;
  static DofPartition from_names(std::vector<std::string> order, const std::vector<std::string>& names);
  Index field_id(const std::string& name) const;
};
void split(const DofPartition& p, const std::vector<std::string>& f_fields, IndexList& F, IndexList& C);

enum class InterpKind { ideal, jacobi };
enum class RestrictKind { injection, jacobi, ideal };

Csr build_interp(const Csr& A, const IndexList& F, const IndexList& C, InterpKind kind,
                 const BlockLayout* ff_layout = nullptr);             // mgr.cpp:89-114
Csr build_restrict(const Csr& A, const IndexList& F, const IndexList& C, RestrictKind kind,
                   const BlockLayout* ff_layout = nullptr);           // mgr.cpp:116-146
Csr coarse_operator(const Csr& A, const Csr& R, const Csr& P);        // mgr.cpp:148-152
Csr schur_jacobi_direct(const Csr& A, const IndexList& F, const IndexList& C);  // 154-165

struct CoarseSolverSpec {
  enum class Kind { dense_lu, amg_vcycle, gmres_inner };
  Kind kind = Kind::dense_lu;
  AmgConfig amg;
  Index amg_cycles = 1;
  bool use_unknown_map = false;
  KrylovConfig krylov;
};

struct MgrLevelSpec {
  std::vector<std::string> f_fields;
  InterpKind interp = InterpKind::jacobi;
  RestrictKind restrict_kind = RestrictKind::injection;
  SmootherSpec f_relax;
  std::optional<SmootherSpec> global_relax;
  std::optional<std::vector<Index>> ff_block_sizes;
};

struct MgrStrategy {
  std::string name;
  std::vector<MgrLevelSpec> levels;
  CoarseSolverSpec coarse;
};

struct MgrLevel {
  Csr A;
  IndexList F, C;
  Csr P, R;
  BoundSmoother f_relax;
  std::optional<BoundSmoother> global_relax;
  IndexList finest_ids;
};

struct MgrHierarchy {
  std::vector<MgrLevel> levels;
  Csr A_coarse;
  CoarseSolverSpec coarse_spec;
  DenseLU coarse_lu;
  std::shared_ptr<AmgHierarchy> coarse_amg;
  IndexList coarse_finest_ids;
  std::vector<int> coarse_unknown_map;
  Index num_reduction_levels() const { return static_cast<Index>(levels.size()); }
  Index fine_size() const { return levels.empty() ? A_coarse.rows : levels.front().A.rows; }
};

MgrHierarchy mgr_setup(const Csr& A, const DofPartition& partition, const MgrStrategy& strategy,
                       const std::vector<int>* unknown_map = nullptr);  // mgr.cpp:223-316
Vec mgr_apply(const MgrHierarchy& H, const Vec& v);                     // mgr.cpp:318-321
LinOp mgr_preconditioner(const MgrHierarchy& H);                        // mgr.cpp:323-326

// ---- strategy JSON (proj/src/strategy_json.cpp) ----------------------------
MgrStrategy strategy_from_json_text(const std::string& text);
std::string strategy_to_json_text(const MgrStrategy& s);

}  // namespace refcpu
