// Single-CTA AMG tail: the coarsest levels of a V-cycle (whose operators,
// transfers, smoother diagonals and coarsest LU factors together fit in one
// SM's shared memory) executed by ONE kernel launch with everything resident
// on chip. The same per-row sequential arithmetic as the launch-per-operation
// V-cycle (amg.cpp:232-242 via AmgHier::vcycle_level), so results are
// bitwise equal; it replaces ~7 launch-latency-bound kernels per tail level
// plus the coarsest dense solve.
#pragma once

#include <vector>

#include "common.cuh"

namespace mgrx {

constexpr int kTailMaxLevels = 6;

struct TailLevel {
  int m = 0, mc = 0;                    // rows of this level / of the next one
  int a_ptr = 0, a_col = 0, a_val = 0;  // byte offsets into the blob
  int r_ptr = 0, r_col = 0, r_val = 0;
  int p_ptr = 0, p_col = 0, p_val = 0;
  int dpre = 0, dpost = 0;              // smoother inverse (l1-)diagonals
  int pre_sweeps = 0, post_sweeps = 0;
  double pre_w = 1.0, post_w = 1.0;
  int vr = 0, vz = 0, vt = 0, v1 = 0, v2 = 0;  // work vectors (byte offsets)
  // cluster tail only: per-CTA row chunk tables of A / R / P (byte offsets)
  int a_chunks = 0, r_chunks = 0, p_chunks = 0;
};

struct TailDesc {
  int nlev = 0;                 // smoothed levels in the tail (the coarsest follows)
  TailLevel L[kTailMaxLevels];
  int nc = 0, lu = 0, perm = 0, cr = 0, cz = 0;  // coarsest dense system
  int blob_bytes = 0, total_bytes = 0;           // blob (copied in) + work vectors
};

// Host-side builder input: one smoothed level of the tail.
struct TailLevelHost {
  int m = 0, mc = 0;
  std::vector<int> a_ptr, a_col, r_ptr, r_col, p_ptr, p_col;
  std::vector<double> a_val, r_val, p_val, dpre, dpost;
  int pre_sweeps = 1, post_sweeps = 1;
  double pre_w = 1.0, post_w = 1.0;
};

// Pack levels + coarsest LU (column-major nc x nc, perm) into a blob; returns
// false when it does not fit in max_bytes of shared memory.
bool build_tail_blob(const std::vector<TailLevelHost>& lv, int nc, const std::vector<double>& lu,
                     const std::vector<int>& perm, size_t max_bytes, TailDesc& d, std::vector<unsigned char>& blob);
// z = V-cycle tail(r): r, z have d.L[0].m entries.
void launch_amg_tail(const TailDesc& d, const unsigned char* blob, const double* r, double* z, cudaStream_t s);
void prepare_amg_tail(const TailDesc& d);

// Cluster AMG tail: the same V-cycle tail run by ONE thread-block cluster of
// kCtCtas CTAs for levels too large for a single CTA (up to kCtMaxRows rows):
// the operators stay in global memory (L2 after their first pass), CTA c owns a
// contiguous row slice of every level, the vector an operator gathers from is
// replicated in every CTA's shared memory (each CTA pushes its slice to its
// peers through distributed shared memory) and a cluster barrier separates the
// operations. Row sums are formed exactly as in the launch-per-operation path
// (products in entry order, summed left to right), so results are bitwise equal.
constexpr int kCtCtas = 16;       // CTAs in the cluster (non-portable size)
constexpr int kCtThreads = 512;
constexpr int kCtProd = 8192;     // products per chunk (64 KB of shared memory)
constexpr int kCtMaxChunks = 16;  // row chunks per CTA and operator
constexpr int kCtMaxRows = 8192;  // largest level
// Pack levels into a global-memory blob with the per-CTA chunk tables; false
// when a level is too large for the shared-memory layout.
// Shared-memory layout of the cluster tail (byte offsets, the same in every
// CTA). Per operator: the CTA's chunk table and its slice of the row
// pointers are always resident; the slice's column indices / values too when
// they fit (col >= 0), otherwise they are read from global memory.
struct CtMat {
  int ptr = 0, chunks = 0, col = -1, val = -1;
};
struct CtLayout {
  int full0 = 0, full1 = 0, prod = 0;
  int vr[kTailMaxLevels + 1] = {}, vz[kTailMaxLevels] = {}, vt[kTailMaxLevels] = {}, vv[kTailMaxLevels] = {};
  CtMat A[kTailMaxLevels], R[kTailMaxLevels], P[kTailMaxLevels];
  int dpre[kTailMaxLevels] = {}, dpost[kTailMaxLevels] = {};  // smoother diagonals, slice-local
  int total = 0;
};
bool build_ctail_blob(const std::vector<TailLevelHost>& lv, int nc, const std::vector<double>& lu,
                      const std::vector<int>& perm, TailDesc& d, std::vector<unsigned char>& blob, CtLayout& lay);
void prepare_amg_ctail(const CtLayout& lay);
void launch_amg_ctail(const TailDesc& d, const CtLayout& lay, const unsigned char* blob, const double* r, double* z,
                      cudaStream_t s);

}  // namespace mgrx
