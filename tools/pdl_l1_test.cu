// Does griddepcontrol.wait make a prerequisite grid's writes visible to
// L1-cached (ld.global.nc / plain ld.global) loads when the dependent grid's
// CTAs became resident early (launch_dependents at entry)?
//
// Chain per round: A reads X through L1 for a while (caching its lines on
// every SM) after signalling its dependents at entry; B (dependent of A)
// signals at entry, waits, then rewrites X; C (dependent of B) signals at
// entry, waits, then reads X with __ldg and counts values that are not B's.
// With entry signals C's CTAs can be resident (and the launch-time L1
// invalidation long past) while A is still filling L1 with the old X. A stale
// count of 0 over many rounds says the wait invalidates (acquires) L1.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pdl_l1_test tools/pdl_l1_test.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      std::printf("CUDA error %s at %d\n", cudaGetErrorString(e_), __LINE__); \
      std::exit(1);                                                            \
    }                                                                          \
  } while (0)

__global__ void kA(const double* __restrict__ x, int n, int reps, double* sink) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  double s = 0.0;
  for (int r = 0; r < reps; ++r)
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += __ldg(x + ((i * 17 + r * 5 + blockIdx.x) % n));
  if (s == 123.456) sink[0] = s;
}
__global__ void kB(double* x, int n, double v) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) x[i] = v;
}
__global__ void kC(const double* __restrict__ x, int n, double v, unsigned long long* bad) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // touch x's neighbourhood before the wait? no: only after (the product rule)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  unsigned long long b = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) b += __ldg(x + ((i * 13 + blockIdx.x) % n)) != v;
  if (b) atomicAdd(bad, b);
}

template <class... KArgs, class... Args>
void launch(void (*k)(KArgs...), int grid, int block, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...));
}

int main() {
  const int n = 4096;  // 32 KB: stays in every SM's L1
  double *x, *sink;
  unsigned long long* bad;
  CK(cudaMalloc(&x, n * sizeof(double)));
  CK(cudaMalloc(&sink, sizeof(double)));
  CK(cudaMalloc(&bad, sizeof(unsigned long long)));
  CK(cudaMemset(bad, 0, sizeof(unsigned long long)));
  CK(cudaMemset(x, 0, n * sizeof(double)));
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  const int rounds = 2000;
  for (int r = 0; r < rounds; ++r) {
    const double v = 1.0 + r;
    // A: 1 CTA per SM at 128 threads (leaves room for B's and C's CTAs)
    launch(kA, 148, 128, s, static_cast<const double*>(x), n, 4 + (r % 7), sink);
    launch(kB, 148, 128, s, x, n, v);
    launch(kC, 148 * 2, 128, s, static_cast<const double*>(x), n, v, bad);
  }
  CK(cudaStreamSynchronize(s));
  unsigned long long h = 0;
  CK(cudaMemcpy(&h, bad, sizeof h, cudaMemcpyDeviceToHost));
  std::printf("pdl_l1_test: rounds %d stale values %llu -> %s\n", rounds, h, h ? "STALE L1 READS" : "ok");
  return h ? 2 : 0;
}
