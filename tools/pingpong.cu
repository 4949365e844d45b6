// Microbenchmark: cross-SM hand-off latency through L2 with relaxed
// gpu-scope stores/loads (the primitive of the sync-free GS sweep).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double ldr(const double* p) { double v; asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p)); return v; }
__device__ __forceinline__ void str(double* p, double v) { asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" :: "l"(p), "d"(v)); }
__device__ __forceinline__ double ldv(const volatile double* p) { return *p; }
// CTA 0 and CTA 1 alternate: CTA b waits for value k (written by the other), writes k+1.
__global__ void pingpong(double* buf, int iters, int mode, long long* cyc, int sleepns) {
  if (threadIdx.x != 0) return;
  const int me = blockIdx.x;
  long long t0 = clock64();
  for (int k = me; k < iters; k += 2) {
    const double want = (double)k;
    if (k > 0) {
      while (true) {
        double v = mode == 0 ? ldr(buf) : ldv(buf);
        if (v >= want) break;
        if (sleepns) __nanosleep(sleepns);
      }
    }
    if (mode == 0) str(buf, want + 1.0); else *(volatile double*)buf = want + 1.0;
  }
  cyc[me] = clock64() - t0;
}
int main() {
  double* buf; long long* cyc;
  cudaMalloc(&buf, 8 * 64); cudaMalloc(&cyc, 16);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int mode = 0; mode < 2; ++mode)
    for (int sl : {0, 20, 100}) {
      cudaMemset(buf, 0, 8);
      const int iters = 20000;
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      pingpong<<<2, 32>>>(buf, iters, mode, cyc, sl);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("mode=%s sleep=%d: %.3f us per hand-off (err=%s)\n", mode ? "volatile" : "relaxed.gpu", sl,
             ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
