// Microbenchmark: cross-SM hand-off latency through distributed shared memory
// (a 2-CTA cluster; the producer stores into the consumer's shared memory with
// st.shared::cluster, the consumer polls its own shared memory), against the
// L2 hand-off of tools/pingpong.cu. Gauge for a cluster-resident Gauss-Seidel
// sweep (dependency hops through DSMEM instead of L2).
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__global__ void __cluster_dims__(2, 1, 1) pingpong_dsmem(int iters, long long* cyc, int chain) {
  __shared__ double slot;
  cg::cluster_group cl = cg::this_cluster();
  const unsigned me = cl.block_rank();
  if (threadIdx.x == 0) slot = 0.0;
  cl.sync();
  if (threadIdx.x == 0) {
    double* peer = cl.map_shared_rank(&slot, me ^ 1);
    volatile double* mine = &slot;
    long long t0 = clock64();
    for (int k = me; k < iters; k += 2) {
      const double want = (double)k;
      double v = 0.0;
      if (k > 0)
        while ((v = *mine) < want) {
        }
      // `chain` dependent fp64 ops stand in for a row's mul/sub/div chain
      double s = want + 1.0 + 0.0 * v;
      for (int c = 0; c < chain; ++c) s = __dadd_rn(__dmul_rn(s, 1.0), 0.0);
      *reinterpret_cast<volatile double*>(peer) = s;
    }
    cyc[me] = clock64() - t0;
  }
  cl.sync();
}

__device__ __forceinline__ double ldr(const double* p) { double v; asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p)); return v; }
__device__ __forceinline__ void str(double* p, double v) { asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" :: "l"(p), "d"(v)); }
__global__ void pingpong_l2(double* buf, int iters, int chain) {
  if (threadIdx.x != 0) return;
  const int me = blockIdx.x;
  for (int k = me; k < iters; k += 2) {
    const double want = (double)k;
    double v = 0.0;
    if (k > 0)
      while ((v = ldr(buf)) < want) {
      }
    double s = want + 1.0 + 0.0 * v;
    for (int c = 0; c < chain; ++c) s = __dadd_rn(__dmul_rn(s, 1.0), 0.0);
    str(buf, s);
  }
}

int main() {
  long long* cyc;
  double* buf;
  cudaMalloc(&cyc, 16);
  cudaMalloc(&buf, 64);
  const int iters = 20000;
  for (int chain : {0, 8}) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    pingpong_dsmem<<<2, 32>>>(64, cyc, chain);
    cudaEventRecord(a);
    pingpong_dsmem<<<2, 32>>>(iters, cyc, chain);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("dsmem  chain=%d: %.3f us per hand-off (err=%s)\n", chain, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    cudaMemset(buf, 0, 8);
    pingpong_l2<<<2, 32>>>(buf, 64, chain);
    cudaMemset(buf, 0, 8);
    cudaEventRecord(a);
    pingpong_l2<<<2, 32>>>(buf, iters, chain);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("l2     chain=%d: %.3f us per hand-off (err=%s)\n", chain, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
