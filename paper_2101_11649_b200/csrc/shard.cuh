// Row-slab sharded MGR-GMRES: one rank per GPU, each owning
// a contiguous row block of every operator at every level.
//
// Setup ("phase 1" of §8e): every rank holds the same global hierarchy (the
// setup kernels are bit-exact, so replicas are identical) and keeps its slab
// of each operator, columns renumbered [owned | halo]. Because every rank
// can read every operator, each rank derives its send lists (what its
// neighbours' rows reference among its columns) without any setup traffic.
// The slab-major dof numbering makes each index space contiguous per rank at
// every level: MGR F/C sets are ascending subsets (proj/src/mgr.cpp:27-35)
// and AMG coarse points keep fine order (proj/src/amg.cpp:209-222), so a
// rank's coarse rows are the C points inside its fine range.
//
// Solve: the single-GPU kernels on the local slabs, with a halo exchange
// (NCCL send/recv) before every product that reads another rank's entries;
// inner products reduce per rank in the canonical order, all-gather the
// per-rank partials and sum them in rank order on the device (every rank
// gets the same bits, run to run). Coarsest dense solves are replicated
// (all-gather of the coarse vector). The preconditioner application is
// bitwise identical to the single-GPU one (same rows, same entry order, same
// arithmetic); only the inner-product reduction order differs.
//
// Smoothers: jacobi, l1_jacobi, amg_vcycle and dense_lu shard exactly. The
// hybrid Gauss-Seidel sweep with one range is sequential over the whole
// matrix and block_jacobi_exact blocks may straddle slabs: both are rejected.
#pragma once

#include <deque>
#include <map>
#include <tuple>
#include <memory>
#include <vector>

#include "comm.hpp"
#include "hierarchy.cuh"
#include "krylov.cuh"

namespace mgrx {

struct Part {
  std::vector<int> st;  // size + 1 starts
  int lo(int r) const { return st[r]; }
  int hi(int r) const { return st[r + 1]; }
  int n(int r) const { return st[r + 1] - st[r]; }
  int total() const { return st.back(); }
  int owner(int g) const;
};

// Index space of one level vector: partition + extended capacity (owned +
// the largest halo any operator reading it needs).
struct Space {
  Part part;
  int own = 0;
  int cap = 0;
  void need(int halo) { cap = cap > own + halo ? cap : own + halo; }
};

// One operator's slab with its halo plan.
struct Seg {
  int peer, off, count;
};
struct SOp {
  DCsr M;  // local rows; columns [0, own) owned, [own, own + nhalo) halo
  int own = 0, nhalo = 0;
  std::vector<Seg> recv;  // off: position in the halo region
  std::vector<Seg> send;  // off: position in sbuf / sidx
  DVec<int> sidx;          // owned column indices to pack, per send segment
  DVec<double> sbuf;
  bool built = false;
};

struct ShardCtx {
  Comm* comm = nullptr;
  cudaStream_t s = nullptr;
  int rank = 0, size = 1;
  bool exact = true;  // false: replicated dense solves through their inverses (low-sync solve)
};

// Replicated dense solve: all-gather the distributed vector, solve on every
// rank with the same factors, keep the own slice.
struct Repl {
  const DenseLU* lu = nullptr;
  Part part;
  int maxc = 0;
  DVec<double> pad, all, full, sol;
  DVec<int> map;
  void build(const DenseLU* f, const Part& p, cudaStream_t s);
  void solve(const double* r, double* z, ShardCtx& c);
};

struct SAmg;

struct SRelax {
  Smoother kind = Smoother::jacobi;
  int sweeps = 1;
  double weight = 1.0;
  int n = 0;
  DVec<double> dinv;
  SOp A;
  std::unique_ptr<SAmg> amg;
  Repl dense;
  Space* sp = nullptr;
  DVec<double> b0, b1, b2, b3;
  void alloc(cudaStream_t s);
  // z = smoother(r[rrow]) (rrow: local gather indices or null); zacc: += instead
  void apply(const double* r, const int* rrow, double* z, double* zacc, ShardCtx& c);
};

struct SAmgLevel {
  Space* sp = nullptr;  // this level's index space
  SOp A, P, R;
  SRelax pre, post;
  DVec<double> r, z, t;
};

// Replicated coarse V-cycle (SURVEY 8(e) agglomeration): from level `from`
// on (<= MGRX_SHARD_REPL_ROWS global rows, Jacobi-type smoothing), every
// rank all-gathers the level's residual and runs the rest of the V-cycle on
// the full vectors with the single-GPU kernels of its own replica of the
// hierarchy (read-only) and shard-owned work vectors, then keeps its slice:
// one all-gather replaces a halo exchange per operation on the small levels.
// The operations are the single-GPU V-cycle's, so results stay bitwise.
struct RepAmg {
  const AmgHier* g = nullptr;
  int from = -1;  // first replicated level of g
  int at = -1;    // the sharded AMG level it replaces (-1: none)
  Part part;  // partition of level `from`
  int maxc = 1;
  DVec<double> pad, all, rfull, zfull;
  DVec<int> map;
  struct Lv {
    DVec<double> r, z, t, w1, w2;
  };
  std::deque<Lv> lv;  // levels from .. coarsest
  void build(const AmgHier& h, int l, const Part& p, cudaStream_t s);
  void vcycle(const double* r, double* z, ShardCtx& c);  // r, z: owned slices of level `from`

 private:
  void level(int l, const double* r, double* z, cudaStream_t s);
  void smooth(const BoundRelax& b, const double* r, double* z, double* zacc, Lv& w, cudaStream_t s);
};

struct SAmg {
  std::deque<Space> spaces;  // spaces[0] unused when the fine space is external
  std::deque<SAmgLevel> L;
  Repl coarse;
  RepAmg rep;  // rep.at >= 1: levels from rep.at on are replicated
  void alloc(cudaStream_t s);
  void vcycle(const double* r, double* z, ShardCtx& c) { level(0, r, z, c); }

 private:
  void level(int l, const double* r, double* z, ShardCtx& c);
};

struct SMgrLevel {
  Space* sl = nullptr;  // level space
  Space* sf = nullptr;  // F space
  Space* sc = nullptr;  // C space (= next level space)
  bool injection = true, general = false;
  int nl = 0, nf = 0, nc = 0;
  DVec<int> Floc, Cloc, fpos;  // local F / C rows, F position of each local row
  SOp A, P, R, Acf;
  SRelax f_relax;
  std::unique_ptr<SRelax> g_relax;
  DVec<double> zF, rc, e, t, vF;
};

struct Shard {
  ShardCtx c;
  std::unique_ptr<Comm> comm;
  std::deque<Space> spaces;  // [0] fine level
  std::deque<SMgrLevel> levels;
  SOp Afine;  // the GMRES operator
  SOp Acoarse;
  Repl coarse_lu;
  std::unique_ptr<SAmg> coarse_amg;
  int coarse_cycles = 1;
  DVec<double> ct, cd;
  // GMRES work (owned rows; x and z with the fine space's halo capacity)
  GmresWork ws;
  DVec<double> xext, zext, loc, gbuf;
  int row_begin = 0, row_end = 0;
  std::map<std::tuple<const double*, double*, bool>, std::pair<cudaGraphExec_t, long long>> graphs_;

  // replicated small parts this shard owns (dense coarse factors, the
  // coarse AMG levels it replicates), built from the plan's small matrices
  std::deque<DCsr> own_mat;
  std::deque<DenseLU> own_lu;
  std::vector<std::unique_ptr<AmgHier>> own_amg;

  // Every rank holds the global hierarchy h (a replica): plan, keep own slab.
  // s: the shard's stream (owned by the caller, outlives the shard)
  void build(MgrHier& h, const DCsr& A, const std::vector<int>& fine_starts, std::unique_ptr<Comm> cm,
             cudaStream_t s);
  // Only rank 0 holds the global hierarchy (h, A non-null there, null
  // elsewhere): it plans for every rank and sends each its plan
  // (shardplan.cu). No global operator ever lives on the other ranks.
  void build_scatter(MgrHier* h, const DCsr* A, const std::vector<int>& fine_starts, std::unique_ptr<Comm> cm,
                     cudaStream_t s);
  void load(const std::vector<unsigned char>& plan);
  ~Shard();
  // z = M^{-1} v on the owned rows (device pointers; z needs no halo room)
  void apply(const double* v, double* z);
  GmresResult solve(const double* b, double* x, const KrylovSpec& cfg);
  GmresResult solve_lowsync(const double* b, double* x, const KrylovSpec& cfg);

  // Fused sharded Arnoldi (krylov.cu arnoldi_sharded): each GMRES step's
  // whole MGS in one kernel per rank, the per-projection rank partials
  // exchanged through IPC-mapped mailboxes over NVLink instead of one
  // all-gather + fold launch pair per projection. Enabled at build when every
  // rank can map every peer and a self-check step equals the all-gather path
  // bit for bit (MGRX_SHARD_FUSED=0: off).
  bool fused = false;
  double* mbox = nullptr;
  std::vector<void*> peer_mbox;
  DVec<double*> peer_dev;
  unsigned long long epoch = 0;

 private:
  void setup_fused();
  ArnoldiPeers peers_arg();
  void apply_level(int l, const double* v, double* z);
  void coarse_solve(const double* v, double* z);
  void prec(const double* v, double* z);
};

}  // namespace mgrx
