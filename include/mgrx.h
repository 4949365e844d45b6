/* mgrx — B200-native MGR-preconditioned GMRES (sm_100a), C ABI.
 *
 * Drop-in boundary for the hot path of the reference mgrkit library
 * (arXiv 2101.11649 reference, /root/reference/proj). The reference exposes a
 * C++ API; each entry point below replaces one of its calls (file:line):
 *
 *   mgrx_matrix_csr  <- SpMat + validate()        proj/include/mgrkit/sparse.hpp:19-22,
 *                                                 proj/src/sparse.cpp:24-41
 *   mgrx_setup       <- mgr_setup(A, partition, strategy, unknown_map)
 *                                                 proj/include/mgrkit/mgr.hpp:105-106
 *                       + strategy_from_json_text proj/include/mgrkit/strategy_json.hpp:11
 *   mgrx_apply       <- mgr_apply(H, v)           proj/include/mgrkit/mgr.hpp:111
 *   mgrx_solve       <- gmres(A, b, x, cfg, mgr_preconditioner(H))
 *                                                 proj/include/mgrkit/krylov.hpp:33-34,
 *                                                 proj/include/mgrkit/mgr.hpp:114
 *   mgrx_solve_op    <- the same call with A != H's fine operator (hierarchy
 *                       kept across Newton steps)
 *   mgrx_spmv        <- spmv(A, x)                proj/include/mgrkit/sparse.hpp:57
 *   mgrx_dump        <- MgrHierarchy / AmgHierarchy member access (levels[l].P, ...)
 *                                                 proj/include/mgrkit/mgr.hpp:79-100,
 *                                                 proj/include/mgrkit/amg.hpp:26-49
 *   mgrx_last_error  <- the what() text of the exception the reference throws
 *
 * Status codes mirror the CLI exit codes (proj/tools/mgr_main.cpp:34):
 *   MGRX_OK 0, MGRX_NOT_CONVERGED 1, MGRX_INVALID_ARGUMENT 2 (std::invalid_argument),
 *   MGRX_RUNTIME 3 (std::runtime_error / logic_error / CUDA failures).
 *
 * Ownership: the library owns all device memory; the caller owns every host
 * buffer it passes. Matrices are copied at creation (the reference copies
 * into the hierarchy, proj/src/mgr.cpp:257). Handles are not thread-safe;
 * each context runs on one CUDA stream. A built hierarchy is immutable.
 * Indices are int32 and values fp64, as in proj/include/mgrkit/types.hpp:17-20.
 */
#ifndef MGRX_H
#define MGRX_H

#if defined(__GNUC__)
#define MGRX_API __attribute__((visibility("default")))
#else
#define MGRX_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define MGRX_OK 0
#define MGRX_NOT_CONVERGED 1
#define MGRX_INVALID_ARGUMENT 2
#define MGRX_RUNTIME 3

typedef struct mgrx_ctx mgrx_ctx;
typedef struct mgrx_mat mgrx_mat;
typedef struct mgrx_hier mgrx_hier;

/* KrylovConfig, proj/include/mgrkit/krylov.hpp:14-19, plus the choice of
 * orthogonalisation (a zero-initialised struct gets the default):
 *   MGRX_ORTHO_DEFAULT / MGRX_ORTHO_CGS2  low-synchronisation lagged CGS2
 *       (two basis sweeps and two reductions per step, device-resident
 *       restart cycle); matches the reference to the north_star bar
 *       (history 1e-10 relative, iterations +-1);
 *   MGRX_ORTHO_MGS  the reference's modified Gram-Schmidt with conditional
 *       re-orthogonalisation (proj/src/krylov.cpp:80-101), bitwise
 *       reproducible against the CPU oracle. */
#define MGRX_ORTHO_DEFAULT 0
#define MGRX_ORTHO_MGS 1
#define MGRX_ORTHO_CGS2 2
typedef struct mgrx_krylov {
  int restart;
  int max_iters;
  double rel_tol;
  double abs_tol;
  int ortho;
} mgrx_krylov;

/* SolveReport, proj/include/mgrkit/krylov.hpp:21-28, plus timings. The
 * history holds one Arnoldi estimate per inner step and the true relative
 * residual after each restart (same layout as the reference). */
typedef struct mgrx_report {
  int converged;
  int iterations;
  double final_residual;
  double* history;   /* caller buffer, may be NULL */
  int history_cap;
  int history_len;   /* full length, may exceed history_cap */
  double setup_s;    /* hierarchy build time (device events) */
  double solve_s;    /* solve time (device events, host copies excluded) */
  long long gpu_launches; /* kernels launched by this call */
} mgrx_report;

/* Thread-local message of the last failing call on this thread. */
MGRX_API const char* mgrx_last_error(void);

/* devices: CUDA ordinals; this build drives devices[0] (one process per GPU). */
MGRX_API int mgrx_create(const int* devices, int ndev, mgrx_ctx** out);
MGRX_API int mgrx_destroy(mgrx_ctx* ctx);
/* Device memory of the context's GPU held by libmgrx (stream-ordered pool):
 * bytes in use now, reserved by the pool, and the in-use high-water mark. */
MGRX_API int mgrx_device_memory(mgrx_ctx* ctx, long long* used, long long* reserved, long long* high);

/* CSR with sorted, in-range columns and finite values (validate()). host
 * pointers; copied to HBM. */
MGRX_API int mgrx_matrix_csr(mgrx_ctx* ctx, int rows, int cols, const int* rowptr, const int* colidx,
                    const double* values, mgrx_mat** out);
/* Same, from pointers that already live in device memory of ctx's GPU. */
MGRX_API int mgrx_matrix_csr_device(mgrx_ctx* ctx, int rows, int cols, const int* d_rowptr,
                           const int* d_colidx, const double* d_values, mgrx_mat** out);
MGRX_API int mgrx_matrix_destroy(mgrx_mat* m);

/* y = A x. flags: bit 0 (MGRX_ON_DEVICE, value 1) x, y are device pointers;
 * bit 2 (MGRX_TEAM_SUMS, value 4) allow the matrix's team-sum kernel, if the
 * setup timing chose one (rows summed by a lane team with fused multiply-adds
 * and a shuffle tree: tolerance-level, what the default solve runs).
 * Without it the row sums are the reference's left-to-right sums (Eigen's
 * y = A*x), bitwise. */
#define MGRX_TEAM_SUMS 4
MGRX_API int mgrx_spmv(mgrx_mat* m, const double* x, double* y, int flags);

/* Build the MGR hierarchy on the GPU. labels[i] in [0, nfields) names
 * field_names[labels[i]] (DofPartition, proj/include/mgrkit/mgr.hpp:20-28).
 * unknown_map may be NULL. strategy_json uses the reference schema
 * (proj/src/strategy_json.cpp:75-228); unknown keys are errors. */
MGRX_API int mgrx_setup(mgrx_ctx* ctx, mgrx_mat* A, const int* labels, int nfields,
               const char* const* field_names, const int* unknown_map, const char* strategy_json,
               mgrx_hier** out);
MGRX_API int mgrx_hier_destroy(mgrx_hier* h);

/* z = M^{-1} v, one MGR V-cycle from zero (mgr_apply). */
MGRX_API int mgrx_apply(mgrx_hier* h, const double* v, double* z, int on_device);

/* Right-preconditioned restarted GMRES with M = mgr_apply (gmres()). x holds
 * the initial guess on entry and the solution on exit. Returns MGRX_OK or
 * MGRX_NOT_CONVERGED (report filled in both cases).
 * flags: bit 0 (MGRX_ON_DEVICE) b and x are device pointers (else host; use
 * pinned host memory for full copy bandwidth); bit 1 (MGRX_ZERO_GUESS) the
 * initial guess is zero and x is not read (no host->device copy of x). */
#define MGRX_ON_DEVICE 1
#define MGRX_ZERO_GUESS 2
MGRX_API int mgrx_solve(mgrx_hier* h, const double* b, double* x, const mgrx_krylov* cfg,
               mgrx_report* report, int flags);

/* The same GMRES with a caller's operator A (square, as many rows as the
 * hierarchy's fine level) and the hierarchy h as M: gmres(A, b, x, cfg,
 * mgr_preconditioner(H)) with A != H.levels[0].A, proj/include/mgrkit/
 * krylov.hpp:33-34 takes the two separately. This is the reuse of a
 * hierarchy across Newton steps (the reference's Newton
 * driver, proj/src/problems/mfd.cpp:650-677, rebuilds it every step): build
 * A_k with mgrx_matrix_csr / mgrx_matrix_csr_device, keep h from an earlier
 * step. Errors as the reference's: "gmres: matrix must be square",
 * "mgr_apply: size mismatch". A and h must belong to one context. */
MGRX_API int mgrx_solve_op(mgrx_hier* h, mgrx_mat* A, const double* b, double* x, const mgrx_krylov* cfg,
                           mgrx_report* report, int flags);

/* AmgSetupInfo of an AMG hierarchy (proj/include/mgrkit/amg.hpp:35-39):
 * which = -1 the MGR coarse solver's AMG, l >= 0 the F-relaxation AMG of MGR
 * level l. level_sizes receives up to cap sizes (nlevels = full count);
 * fallback_rows = interpolation rows on the diagonally scaled fallback
 * (proj/src/amg.cpp:115-122); truncated = coarsening stalled. */
MGRX_API int mgrx_amg_info(mgrx_hier* h, int which, int* nlevels, int* level_sizes, int cap,
                           long long* fallback_rows, int* truncated);

/* Negative control (proj/src/verify.cpp:105-134, `mgrkit verify
 * --corrupt-transfer`, proj/tests/test_acceptance.cpp:25-30): scales the
 * interpolation P of MGR level `level` by `factor` in place (the reference
 * uses 1.01), so that an exactness check that must then fail can prove it
 * notices. The hierarchy stays usable; there is no undo. */
MGRX_API int mgrx_corrupt_transfer(mgrx_hier* h, int level, double factor);

/* Parity dumps. path grammar:
 *   mgr.<l>.{A,P,R,F,C,frelax.dinv}   mgr.coarse.A
 *   mgr.<l>.frelax.amg.<k>.{A,P,R,C,F,l1d,dinv,umap}   mgr.coarse.amg.<k>.{...}
 * Two-call protocol: pass NULL buffers to query kind/sizes.
 * kind: 0 = CSR (ptr/col/val), 1 = int list (col), 2 = fp64 vector (val). */
MGRX_API int mgrx_dump(mgrx_hier* h, const char* path, int* kind, int* rows, int* cols, long long* nnz,
              int* ptr, int* col, double* val);

/* Hierarchy shape for iterating dumps. frelax_amg_levels has room for
 * max_levels entries. */
MGRX_API int mgrx_info(mgrx_hier* h, int* mgr_levels, int* coarse_amg_levels, int* frelax_amg_levels,
              int max_levels);

/* Roofline probe: replay one hot kernel of the hierarchy `reps` times back
 * to back with its inputs resident in HBM (MGRX_PROBE_FLUSH=1: each launch
 * after a 256 MB L2 flush) and report its average device time (CUDA events
 * on the library stream) and its algorithmic bytes per launch (SURVEY §8d
 * compulsory-traffic model). which:
 *   "spmv.A"            y = A x on the fine matrix (GMRES operator)
 *   "mgr.<l>.rres"      restricted residual v_C - A_CF z_F of MGR level l
 *   "mgr.<l>.prolong"   fused prolongation z = [zF;0] + P e of MGR level l
 *   "amg.<k>.resid"     t = r - A z on level k of the coarse AMG
 *   "amg.<k>.pre"       pre-smoother sweep on level k of the coarse AMG
 *   "amg.<k>.post"      post-smoother sweep on level k of the coarse AMG */
MGRX_API int mgrx_time_kernel(mgrx_hier* h, const char* which, int reps, double* avg_ms,
                              double* bytes);

/* ---- Row-slab sharded solve (one rank per GPU) ----------
 * The reference is single-process (proj/src/krylov.cpp:37-147 over
 * proj/src/mgr.cpp:196-219); these calls distribute that same solve over
 * ranks that each hold the same hierarchy (built by mgrx_setup on every
 * rank) and own a contiguous block of fine rows; coarse levels follow (the
 * C points inside each rank's range). Halo exchanges and the inner-product
 * all-gathers run over NCCL (libnccl.so.2 is loaded at the first NCCL call),
 * or, for tests, between ranks that are threads of one process sharing a
 * "local group". Collective semantics: every rank of a group makes the same
 * sequence of shard calls. */
typedef struct mgrx_shard mgrx_shard;
typedef struct mgrx_group mgrx_group;

/* ncclGetUniqueId; rank 0 calls it and distributes the 128 bytes. */
MGRX_API int mgrx_nccl_unique_id(unsigned char* out128);
/* In-process ranks (threads on one device) for parity tests. */
MGRX_API int mgrx_local_group_create(int size, mgrx_group** out);
MGRX_API int mgrx_local_group_destroy(mgrx_group* g);
/* Bring-your-own transport: the ranks are processes (one per GPU, or several
 * sharing one GPU) connected by the caller's communicator -- MPI in the
 * paper's setting (hypre runs MGR over MPI), gloo in this
 * repo's tests. libmgrx stages every halo segment / all-gather operand
 * through pinned host memory and calls these BLOCKING functions (0 = ok):
 *   exchange: send send_count[i] doubles at send_buf[i] to rank send_peer[i]
 *             for i < nsend and receive recv_count[j] doubles from rank
 *             recv_peer[j] into recv_buf[j] for j < nrecv; every rank calls it
 *             with matching lists, so it must not depend on the order of the
 *             peers' calls (post the receives first / nonblocking sends);
 *   allgather: out[q * count + i] = rank q's in[i].
 * Every rank creates its own group object of the same size and passes it as
 * `group` to mgrx_shard_create[_scatter]; destroy it with
 * mgrx_local_group_destroy after the shard. No reference counterpart (the
 * reference is single-process). */
typedef struct mgrx_transport {
  void* user;
  int (*exchange)(void* user, int nsend, const int* send_peer, const double* const* send_buf, const int* send_count,
                  int nrecv, const int* recv_peer, double* const* recv_buf, const int* recv_count);
  int (*allgather)(void* user, const double* in, double* out, int count);
} mgrx_transport;
MGRX_API int mgrx_transport_group_create(int size, const mgrx_transport* t, mgrx_group** out);
/* row_starts: size+1 fine-row offsets (NULL = even split). Exactly one of
 * nccl_id / group when size > 1. */
MGRX_API int mgrx_shard_create(mgrx_hier* h, int rank, int size, const int* row_starts,
                               const unsigned char* nccl_id, mgrx_group* group, mgrx_shard** out);
/* Scattered setup (SURVEY §8(e) "build on GPU 0, then scatter"): rank 0
 * passes the global hierarchy it built (h), every other rank passes NULL and
 * never holds a global operator. Rank 0 cuts every rank's slabs and halo
 * plans and sends each rank its plan; small replicated parts (dense coarse
 * factors, replicated coarse AMG levels) are rebuilt on each rank from their
 * (small) matrices with the same bit-exact setup. row_starts are required
 * (size+1 fine-row offsets, the same on every rank). After return rank 0 may
 * destroy h; the shard does not reference it. Collective over the group. */
MGRX_API int mgrx_shard_create_scatter(mgrx_ctx* ctx, mgrx_hier* h, int rank, int size, const int* row_starts,
                                       const unsigned char* nccl_id, mgrx_group* group, mgrx_shard** out);
MGRX_API int mgrx_shard_rows(mgrx_shard* sd, int* row_begin, int* row_end);
/* Device bytes allocated while building the hierarchy / this rank's shard
 * (the setup footprint; the GMRES basis is allocated at the first solve). */
MGRX_API int mgrx_hier_bytes(mgrx_hier* h, long long* bytes);
MGRX_API int mgrx_shard_bytes(mgrx_shard* sd, long long* bytes);
/* 1 when this shard's GMRES steps use the fused sharded Arnoldi kernel
 * (in-kernel partial exchange over NVLink; enabled after a bitwise
 * self-check on every rank), 0 for the all-gather path. No reference
 * counterpart (the reference is single-process). */
MGRX_API int mgrx_shard_fused(mgrx_shard* sd, int* fused);
/* z = M^{-1} v on the owned rows (bitwise equal to the owned rows of mgrx_apply). */
MGRX_API int mgrx_shard_apply(mgrx_shard* sd, const double* v, double* z, int on_device);
/* GMRES on the owned rows of b / x (flags as mgrx_solve). */
MGRX_API int mgrx_shard_solve(mgrx_shard* sd, const double* b, double* x, const mgrx_krylov* cfg,
                              mgrx_report* report, int flags);
MGRX_API int mgrx_shard_destroy(mgrx_shard* sd);

#ifdef __cplusplus
}
#endif
#endif /* MGRX_H */
