// Classical AMG coarsening kernels (bit-exact restatements of
// proj/src/amg.cpp:11-141): strength pattern, deterministic PMIS, direct
// interpolation.
#pragma once

#include "sparse.cuh"

namespace mgrx {

// Pattern of strong couplings (values 1.0), proj/src/amg.cpp:11-34.
DCsr strength_graph(const DCsr& A, double theta, cudaStream_t s);

// PMIS C/F splitting on S + S^T with in-degree measure; is_c[i] = 1 for C.
// Returns the number of selection rounds. proj/src/amg.cpp:36-86.
int pmis(const DCsr& S, DVec<uint8_t>& is_c, cudaStream_t s);

// Direct interpolation, proj/src/amg.cpp:88-141. cid[i] = coarse index of C
// point i (or -1). Adds the fallback-row count to *fallback.
DCsr classical_interp(const DCsr& A, const DCsr& S, const int* cid, int nc, long long* fallback,
                      cudaStream_t s);

// cid[i] = rank of i among flagged points, -1 otherwise; returns the count.
int rank_flags(const uint8_t* flag, int n, DVec<int>& cid, cudaStream_t s);

}  // namespace mgrx
