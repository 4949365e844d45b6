// Smoother kernels: pointwise Jacobi/l1-Jacobi and the exact, sync-free
// Gauss-Seidel sweep (proj/src/relax.cpp:55-78 with one range).
#pragma once

#include "sparse.cuh"

namespace mgrx {

// Rows in dependency-level order for one sweep direction: every row's
// dependencies (columns j < i forward, j > i backward) sit at earlier
// positions, which is what makes the sync-free sweep deadlock-free.
struct GsSchedule {
  DVec<int> order;
  int levels = 0;
};
void gs_schedule(const DCsr& A, bool forward, GsSchedule& out, cudaStream_t s);

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
