// Device MGR / AMG hierarchies: setup (bit-exact) and the preconditioner
// application (MGR Algorithm 1, proj/src/mgr.cpp:196-219; AMG V(1,1),
// proj/src/amg.cpp:232-242). All state lives in HBM; the host only sequences
// kernel launches (or replays them from a captured CUDA graph).
#pragma once

#include <deque>
#include <map>
#include <memory>
#include <optional>
#include <string>
#include <tuple>
#include <vector>

#include "amgtail.cuh"
#include "blocklu.cuh"
#include "dense.cuh"
#include "relax.cuh"
#include "strategy.hpp"

namespace mgrx {

struct AmgHier;

// Largest level (rows) whose Jacobi sweep 0 is folded into sweep 1.
int fold_sweep0_max_rows();

// A smoother specialised to one matrix (BoundSmoother, proj/src/relax.cpp:90-192).
struct BoundRelax {
  SmootherSpec spec;
  const DCsr* A = nullptr;  // matrix it is bound to (owned by the enclosing level)
  int n = 0;
  DVec<double> dinv;  // jacobi / l1_jacobi
  DVec<double> l1d;   // gauss-seidel
  GsSchedule sched;
  DVec<int> owner;    // gauss-seidel with a multi-range hybrid partition: range id per row
  BlockLU blk;        // block_jacobi_exact
  std::unique_ptr<AmgHier> amg;
  DenseLU lu;
  DVec<double> w0, w1, w2;  // workspace
  GsScratch gs;

  void bind(const SmootherSpec& s, const DCsr& mat, const std::vector<int>* umap, cudaStream_t st);
  // z = smoother(r) from a zero start; r gathered through rrow when non-null.
  void apply(const double* r, const int* rrow, double* z, cudaStream_t st);
  // Same, but fused accumulate: zacc += smoother(r). r contiguous.
  void apply_add(const double* r, double* zacc, cudaStream_t st);
  void jacobi_sweeps(const double* rc, const int* rrow, double* z, double* zacc, cudaStream_t st,
                     bool have_z0 = false);
  // Jacobi with >= 2 sweeps on a level too large for the folded first sweep:
  // the producer of its input can write sweep 0 into w2 (fused k_jacobi0)
  bool z0_fusable() const;
  void check(cudaStream_t st);
};

struct AmgLevelD {
  DCsr A, P, R;
  std::vector<int> umap;  // unknown id per dof (empty = scalar)
  DVec<int> C, F;         // splitting that produced P (parity dumps)
  BoundRelax pre, post;
  DVec<double> r, z, t;   // level work vectors (r/z unused on level 0)
};

struct AmgHier {
  AmgSpec spec;  // the configuration it was set up with
  std::deque<AmgLevelD> levels;  // deque: smoothers hold pointers to level matrices
  DenseLU coarse;
  std::vector<int> level_sizes;
  long long fallback_rows = 0;
  bool truncated = false;
  // single-CTA tail (amgtail.cuh): levels >= tail run as one kernel; -1: off
  int tail = -1;
  TailDesc tail_desc;
  DVec<unsigned char> tail_blob;
  // cluster tail (amgtail.cuh): levels >= ctail run as one 16-CTA cluster
  // kernel (chosen when it starts above the single-CTA tail); -1: off
  int ctail = -1;
  TailDesc ctail_desc;
  DVec<unsigned char> ctail_blob;
  CtLayout ctail_lay;

  void setup(const DCsr& A, const AmgSpec& cfg, const std::vector<int>& umap, cudaStream_t s);
  void vcycle(const double* r, double* z, cudaStream_t s);
  int fine_size() const { return levels.empty() ? 0 : levels.front().A.rows; }
  void build_tail(cudaStream_t s);
  void build_single_tail(cudaStream_t s);

 private:
  void vcycle_level(int l, const double* r, double* z, cudaStream_t s);
};

// spmv plans and the single-CTA tail of a set-up AMG hierarchy (and of its
// nested smoothers); called once after setup.
void prepare_amg(AmgHier& h, cudaStream_t s);

struct MgrLevelD {
  DCsr A;
  DVec<int> F, C, fpos;
  DCsr P, R, Acf, Aff;
  ProlongPlan pplan;  // split-form prolongation (fast path), w == 0 if unused
  bool injection = true;
  BoundRelax f_relax;
  std::optional<BoundRelax> g_relax;
  DVec<double> zF, rc, e, t, zfull;  // work vectors
};

struct MgrHier {
  std::deque<MgrLevelD> levels;
  DCsr A_coarse;
  CoarseSpec coarse_spec;
  DenseLU coarse_lu;
  std::unique_ptr<AmgHier> coarse_amg;
  DVec<double> ct, cd;  // coarse-cycle work vectors
  int n = 0;

  void setup(const DCsr& A, const std::vector<int>& labels, const std::vector<std::string>& fields,
             const std::vector<int>* umap, const Strategy& strat, cudaStream_t s);
  // exact = false: dense coarse solves through their explicit inverses
  // (tolerance-level; the default solve); exact = true: the bitwise path
  void apply(const double* v, double* z, cudaStream_t s, bool exact = true);
  // z = [0 + zF; 0] + P e of level l (split form when available)
  void prolong(int l, const double* e, const double* zF, double* z, cudaStream_t s);
  // Same, replayed from a CUDA graph captured once per (v, z, exact).
  void apply_graph(const double* v, double* z, cudaStream_t s, bool exact = true);
  // In-situ choice of the x-window SpMV per operator: each candidate plan is
  // switched on / off by timing whole applications (every operator is then
  // read as cold as in the solve, with its real epilogues and neighbours).
  void tune_spmv(cudaStream_t s);
  // Negative control (proj/src/verify.cpp:115, `--corrupt-transfer`): P of
  // MGR level l scaled by `factor` in place; value-holding SpMV copies of P
  // and captured application graphs are dropped so every path sees it.
  void corrupt_transfer(int l, double factor, cudaStream_t s);
  void check(cudaStream_t s);
  ~MgrHier();

 private:
  struct Captured {
    cudaGraphExec_t exec = nullptr;
    long long nodes = 0;
  };
  std::map<std::tuple<const double*, double*, bool>, Captured> graphs_;
  bool exact_dense_ = true;
  void apply_level(int l, const double* v, double* z, cudaStream_t s);
  void coarse_solve(const double* v, double* z, cudaStream_t s);
};

}  // namespace mgrx
