// Smoother kernels: pointwise Jacobi/l1-Jacobi and the exact, sync-free
// Gauss-Seidel sweep (proj/src/relax.cpp:55-78, one range or a hybrid
// partition of ranges).
#pragma once

#include "sparse.cuh"

namespace mgrx {

// Rows in dependency-level order for one sweep direction: every row's
// dependencies (columns j < i forward, j > i backward) sit at earlier
// positions, which is what makes the sync-free sweep deadlock-free.
//
// The schedule also stores the sweep in "sweep CSR" form: rows permuted to
// sweep order, so a CTA's rows are one contiguous block of entries that it
// stages in shared memory with coalesced loads.
//   dep  : only the dependency entries (columns visited earlier in the
//          sweep). A sweep from zero needs nothing else: every other term is
//          a_ij * 0, which leaves the partial sum (and so x_i) unchanged.
//   full : every stored entry, dependency entries flagged by bit 31 of the
//          column (multi-sweep smoothers, whose old iterate is nonzero).
struct GsSchedule {
  DVec<int> order;                 // sweep position -> row
  std::vector<int> level_ptr;      // host: positions of each dependency level
  int levels = 0;
  DVec<int> dptr, dcol;            // dep-only sweep CSR
  DVec<double> dval;
  DVec<int> fptr, fcol;            // full sweep CSR (only when sweeps > 1)
  DVec<double> fval;
  DVec<double> sd;                 // d in sweep order
  bool has_full = false;
  int team = 1;                    // lanes per row in the sync-free kernel
  int cluster = 0;                 // >0: level-synchronous sweep in one cluster of this size
  DVec<int> dlptr;                 // device copy of level_ptr
  int pipe = 0;                    // 1: pipelined single-CTA level sweep
  int small = 0;                   // 1: single-CTA sweep with x in shared memory (n <= 12288)
  DVec<int> dsteps, fsteps;        // step boundaries (positions) for the pipelined sweep
  int ndsteps = 0, nfsteps = 0;
  // single-CTA sweep: groups of consecutive steps loaded together (one
  // cp.async chunk of <= kSmallRows rows / kSmallEnt entries holding many
  // short dependency levels), double-buffered a chunk ahead
  DVec<int> dchunks, fchunks;
  int ndchunks = 0, nfchunks = 0;
  DVec<double> bp;                 // rhs gathered into sweep order (pipelined sweep)
  // Block-partitioned sweep (default for n > 12288, sweeps from zero): the
  // rows are cut into contiguous blocks of <= 12288 (processed in sweep
  // direction); one CTA sweeps a block with its part of the iterate in
  // shared memory, rows in local dependency-level order, so a dependency
  // inside the block costs a barrier; dependencies on earlier blocks are
  // polled from global memory (the value is its own ready flag).
  int blk = 0, nblk = 0;
  DVec<int> blk_lo, blk_chunk;     // per block in processing order: first row, first chunk (nblk + 1)
  DVec<int> border, bsptr, bscol;  // positions in (block, local level) order; dep-only sweep CSR
  DVec<double> bsval, bsd, bbp;    // entry values, d and rhs in that order
  DVec<int> bsteps, bchunks;       // steps (positions, then entry offsets), chunks (step ranges)
  int nbsteps = 0, nbchunks = 0;
};
// owner (nullable): range id per row for a multi-range hybrid partition;
// dependencies are then only the earlier rows of the row's own range.
void gs_schedule(const DCsr& A, bool forward, const double* d, bool full, GsSchedule& out,
                 cudaStream_t s, const int* owner = nullptr);

// Scratch for a GS sweep (ticket counter + error flag).
struct GsScratch {
  DVec<int> ticket_err;  // [0] ticket, [1] error
};

// One exact Gauss-Seidel sweep in sequential semantics:
//   for i in sweep order: s = b_i; for (j,a) in row i: s -= a * x_j; x_i += s / d_i
// where x_j is the new value if j precedes i in the sweep, else the old one.
// xold == nullptr means the sweep starts from zero. xnew receives the result;
// if zadd != nullptr, zadd[i] += xnew[i] is fused in.
void gs_sweep(const DCsr& A, const GsSchedule& sch, const double* d, const double* b,
              const double* xold, double* xnew, double* zadd, bool forward, GsScratch& scr,
              cudaStream_t s);
void gs_bind_scratch(GsScratch& scr, cudaStream_t s);
// Throws if a sweep since the last check hit the spin limit.
void gs_check(GsScratch& scr, cudaStream_t s);

// z = w * (dinv * r), r optionally gathered through rrow (Jacobi sweep 0,
// proj/src/relax.cpp:171). If zadd != nullptr: zadd += that instead of z.
void jacobi0(int n, double w, const double* dinv, const double* r, const int* rrow, double* z,
             cudaStream_t s);

// Pointwise helpers used by the V-cycles.
void vec_add(int n, const double* a, double* y, cudaStream_t s);            // y += a
void gather(int n, const int* idx, const double* x, double* y, cudaStream_t s);  // y = x[idx]
void reciprocal(int n, const double* d, double* y, cudaStream_t s);              // y = 1/d

}  // namespace mgrx
