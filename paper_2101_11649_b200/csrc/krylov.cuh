// Right-preconditioned restarted GMRES on the device
// (proj/src/krylov.cpp:37-147): V, w, x, b in HBM; modified Gram-Schmidt
// with the reference's conditional re-orthogonalisation; deterministic
// fixed-shape reductions; Givens rotations and the small triangular solve on
// the host (O(m^2) scalars per restart).
#pragma once

#include <functional>
#include <memory>
#include <vector>

#include "sparse.cuh"
#include "strategy.hpp"

namespace mgrx {

struct GmresResult {
  bool converged = false;
  int iterations = 0;
  double final_residual = 0.0;
  std::vector<double> history;
};

using DevOp = std::function<void(const double* in, double* out, cudaStream_t s)>;

// Low-synchronisation (lagged CGS2) Arnoldi state, device resident
// (lowsync.cu). flags: stopping reasons of the current restart cycle.
constexpr int kLsConverged = 1, kLsHappy = 2, kLsNonFinite = 4, kLsCycleEnd = 8;
constexpr int kLsMaxRestart = 512;
struct LsState {
  double bnorm, target;
  int k;           // next step index of the cycle (= finalised columns + 1)
  int steps;       // steps done in this cycle
  int iters_left;  // step budget of this cycle
  int flags;
  double gamma, beta;  // last sweep-A normaliser, last preliminary subdiagonal
  double gt0, gt1;     // tentatively rotated g_k, g_{k+1} of the last step
};

struct LsWork {
  int n = 0, m = 0, ldv = 0, G = 0;
  DVec<double> V, U, part, part2, dbl;
  DVec<double> rpart, gath;  // sharded: this rank's sums, all ranks' sums
  DVec<unsigned> ticket;
  DVec<LsState> st;
  LsState* hst = nullptr;  // pinned mirror
  cudaGraphExec_t exec = nullptr;  // one restart cycle (conditional WHILE node)
  struct Key {
    const void* w = nullptr;
    const void* z = nullptr;
    const void* A = nullptr;
  } exec_key;
  long long body_nodes = 0;
  bool graph_failed = false;
  void ensure(int n, int m, cudaStream_t s);
  LsWork() = default;
  LsWork(const LsWork&) = delete;
  LsWork& operator=(const LsWork&) = delete;
  ~LsWork();
};

// Host side of one low-sync GMRES over an LsWork (lowsync.cu), shared by the
// single-GPU solve and the sharded one (shard.cu). The caller runs the
// preconditioner and the SpMV into w from U(), then step()/step_sharded().
struct LsArgs;
class LsDriver {
 public:
  using Allgather = std::function<void(const double* in, double* out, int count, cudaStream_t s)>;
  LsDriver(LsWork& L, int n, int m, double* w);
  ~LsDriver();
  double* U() const;  // the next vector (input of M^-1 each step)
  const LsArgs& args() const;
  void start_cycle(double bnorm, double target, int iters_left, cudaStream_t s);
  void step(cudaStream_t s);  // sweep A + sweep B, single GPU
  // the same with the two reductions completed across ranks: each rank's
  // sums all-gathered and folded in rank order (every rank gets the same bits)
  void step_sharded(int nranks, const Allgather& allgather, cudaStream_t s);
  const LsState& sync_state(cudaStream_t s);
  // end of a restart cycle: appends its residual estimates to hist, y = the
  // triangular solve on the rotated H (empty: nothing to add)
  LsState end_cycle(std::vector<double>& hist, std::vector<double>& y, cudaStream_t s);
  void combine(const std::vector<double>& y, double* u, cudaStream_t s);  // u = V y (synchronises)

 private:
  LsWork& L_;
  int n_, m_;
  double* w_;
  std::unique_ptr<LsArgs> args_;
};

struct GmresWork {
  int n = 0, m = 0;
  DVec<double> V, w, r, z, u;
  DVec<double> scal, part;  // device scalars / reduction partials
  DVec<unsigned> ctr;
  DVec<double> apart;  // fused Arnoldi kernel: double-buffered partials
  DVec<unsigned> bar;  // fused Arnoldi kernel: grid barrier

  std::vector<double> hscal;
  double* hpinned = nullptr;
  LsWork ls;
  void ensure(int n, int m, cudaStream_t s);
  ~GmresWork();
};

// A x = b with x0 in x; all vectors are device pointers. cfg.ortho selects
// the orthogonalisation: kOrthoMgs the reference's MGS (bitwise against the
// oracle), otherwise the lagged CGS2 of lowsync.cu. precond_capture (may be
// empty): the same operator as precond in a form that can be recorded into
// a CUDA graph (no graph launches inside).
GmresResult gmres_device(const DCsr& A, const double* b, double* x, const KrylovSpec& cfg,
                         const DevOp& precond, GmresWork& ws, cudaStream_t s,
                         const DevOp& precond_capture = DevOp());
GmresResult gmres_lowsync(const DCsr& A, const double* b, double* x, const KrylovSpec& cfg,
                          const DevOp& precond, const DevOp& precond_capture, GmresWork& ws, cudaStream_t s);
bool lowsync_supported(int n, int m);
// Probe: the two sweeps of one low-sync step at index k (which: 1 sweep A, 2 sweep B, 3 both).
int lowsync_probe(int n, int k, GmresWork& ws, cudaStream_t s, int which);

// One fused MGS step (w -= h*vprev; a.w) for the roofline probe.
void mgs_probe(int n, double* w, const double* vprev, const double* h, const double* a, GmresWork& ws,
               cudaStream_t s);

// One fused Arnoldi step (both MGS passes in one persistent kernel) on the
// work vectors, for the probe; dbg bits as in ArnoldiArgs. Returns 0 when the
// fused kernel is unavailable for n.
int arnoldi_probe(int n, int k, int dbg, GmresWork& ws, cudaStream_t s);

// Building blocks of the sharded GMRES (shard.cu):
// one MGS kernel on local rows, partial results in out1 / out2 (canonical
// per-rank reduction order); see k_mgs in krylov.cu for the argument roles.
void mgs_step(int n, double* w, const double* vprev, const double* hprev, const double* a, bool want2,
              GmresWork& ws, double* out1, double* hacc, bool accumulate, double* out2, cudaStream_t s);
// out = in / d
void vec_scale(int n, const double* in, double d, double* out, cudaStream_t s);
// u = sum_{j<k} V[j] y[j], j ascending (V column-major, n rows)
void basis_combine(int n, int k, const double* V, const double* y, double* u, cudaStream_t s);

// Sharded fused Arnoldi step (shard.cu): the lane-pair kernel on this rank's
// slab, with every projection's rank partial exchanged through the peers'
// mailboxes (CUDA IPC mappings, stores over NVLink) inside the kernel and
// folded in rank order exactly like the all-gather path's k_fold2. mbox:
// this rank's mailbox (kMboxDoubles doubles, zeroed once); peers: device
// array of every rank's mailbox; epoch: per-launch tag, the same on every
// rank (ranks launch in lockstep). A peer that does not answer within ~2 s
// sets S[m + 3] = 1 (the caller falls back / throws).
constexpr int kMboxRanks = 8, kMboxPhases = 64;
constexpr int kMboxDoubles = kMboxPhases * kMboxRanks * 4;
// published instead of a phase tag once a rank has timed out: every peer
// that reads it flags the step as well
constexpr unsigned long long kMboxPoison = ~0ull;
struct ArnoldiPeers {
  int nranks = 1, rank = 0;
  double* mbox = nullptr;
  double* const* peers = nullptr;
  unsigned long long epoch = 0;
};
bool arnoldi_sharded_ok(int n);
void arnoldi_sharded(int n, int k, int dbg, const ArnoldiPeers& pe, GmresWork& ws, cudaStream_t s);

// Deterministic device dot product (fixed grid, fixed reduction tree).
double device_dot(int n, const double* a, const double* b, GmresWork& ws, cudaStream_t s);

}  // namespace mgrx
