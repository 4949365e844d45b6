// Shared device plumbing for libmgrx: error handling, stream-ordered HBM
// buffers, launch helpers. sm_100a only.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace mgrx {

// Errors mirror the reference's exception split (proj/tools/mgr_main.cpp:492-501):
// InvalidArgument -> status 2, everything else -> status 3.
struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct RuntimeError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define MGRX_CK(x)                                                                             \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess)                                                                     \
      throw ::mgrx::RuntimeError(std::string("CUDA error: ") + cudaGetErrorString(e_) + " (" + \
                                 __FILE__ + ":" + std::to_string(__LINE__) + ")");            \
  } while (0)

#define MGRX_LAUNCH_CK() MGRX_CK(cudaGetLastError())

// NVTX range (header-only NVTX v3; a no-op unless a tool is attached) around
// a phase: setup / application of each MGR and AMG level, the GMRES solve
// (SURVEY §5 tracing). Inside a graph capture the range brackets the capture.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  NvtxRange(const char* what, int level) {
    char buf[48];
    snprintf(buf, sizeof buf, "%s.%d", what, level);
    nvtxRangePushA(buf);
  }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Programmatic dependent launch (PDL): solve-path kernels are launched with
// the programmatic-serialization attribute. griddepcontrol.wait (pdl_wait)
// blocks until the previous grid has completed and its writes are visible
// (it acquires: tools/pdl_l1_test.cu finds no stale L1-cached reads behind
// it). Every access to data a previous kernel may have written comes after
// the wait, so stream order is preserved; what overlaps by default is only
// the launch processing between dependent kernels.
// MGRX_PDL_MODE (compile time) adds early launches, both MEASURED SLOWER and
// therefore off (cfg2 solve, round 2: 54.0 ms without; bit 0 alone 64.2 ms;
// bit 1 alone 57.3 ms; both 62.4 ms): CTAs of an early-launched grid are
// placed greedily on whichever SMs free up first, so the dependent grid
// starts unevenly spread over the SMs and its slowest SM sets its time.
//   bit 0: kernels signal launch_dependents at entry;
//   bit 1: the staged SpMV kernels issue their first stages' bulk copies
//          (matrix data: setup-time constants) before the wait and signal
//          their dependents when a CTA starts its last block.
#ifndef MGRX_PDL_MODE
#define MGRX_PDL_MODE 0
#endif
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_signal() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_enter() {
#if MGRX_PDL_MODE & 1
  pdl_signal();
#endif
  pdl_wait();
}
constexpr bool kPdlStagedEarly = (MGRX_PDL_MODE & 2) != 0;
bool pdl_enabled();

// Under MGRX_PDL_MODE bit 1 only launches flagged `early` (persistent grids
// that fill every SM to their shared-memory limit, so their CTAs cannot pile
// up on the first SMs that drain) may start before the previous grid has
// completed; everything else is then launched fully serialised.
struct PdlEarly {
  bool ok;
};
template <class... KArgs, class... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args);
template <class... KArgs, class... Args>
void launch_pdl(PdlEarly early, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() && (!kPdlStagedEarly || early.ok) ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
  if (e != cudaSuccess)
    throw RuntimeError(std::string("CUDA error: ") + cudaGetErrorString(e) + " (launch grid " +
                       std::to_string(grid.x) + " block " + std::to_string(block.x) + " smem " + std::to_string(smem) +
                       ")");
}
template <class... KArgs, class... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() && !kPdlStagedEarly ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
  if (e != cudaSuccess)
    throw RuntimeError(std::string("CUDA error: ") + cudaGetErrorString(e) + " (launch grid " +
                       std::to_string(grid.x) + " block " + std::to_string(block.x) + " smem " + std::to_string(smem) +
                       ")");
}

// Kernel attributes (dynamic shared memory opt-in, cluster flags) and SM
// counts are per device: one-time setup is keyed by (key, current device),
// so a second context on another GPU in the same process gets its own.
bool first_on_device(const void* key);
int device_sms();  // SM count of the current device (cached per device)
// Raise kernel `kern`'s dynamic shared memory limit on the current device to
// at least `bytes` (never lowers it: several hierarchies in one process size
// the same kernel differently, and the attribute is per kernel, not per launch).
void ensure_smem(const void* kern, size_t bytes);

// Process-wide launch counter (the bench reports kernels launched in the
// timed region; graph replays add their node count).
extern long long g_launches;
inline void count_launch(long long k = 1) { g_launches += k; }

// Device bytes held by DVec allocations made on the calling thread (frees
// are credited to the allocating thread's counter too). Lets a rank that is
// a thread (local groups) measure the footprint of what it built.
long long& thread_device_bytes();

// Stream-ordered device buffer (cudaMallocAsync on the owning stream).
template <class T>
class DVec {
 public:
  DVec() = default;
  DVec(size_t n, cudaStream_t s) { alloc(n, s); }
  DVec(const DVec&) = delete;
  DVec& operator=(const DVec&) = delete;
  DVec(DVec&& o) noexcept { swap(o); }
  DVec& operator=(DVec&& o) noexcept {
    if (this != &o) {
      release();
      swap(o);
    }
    return *this;
  }
  ~DVec() { release(); }

  void alloc(size_t n, cudaStream_t s) {
    release();
    n_ = n;
    s_ = s;
    // +32 bytes: bulk (TMA) copies round slices out to 16-byte multiples
    if (n_) {
      MGRX_CK(cudaMallocAsync(reinterpret_cast<void**>(&p_), n_ * sizeof(T) + 32, s_));
      ctr_ = &thread_device_bytes();
      *ctr_ += static_cast<long long>(n_ * sizeof(T) + 32);
    }
  }
  void release() {
    if (p_) {
      cudaFreeAsync(p_, s_);
      if (ctr_) *ctr_ -= static_cast<long long>(n_ * sizeof(T) + 32);
    }
    p_ = nullptr;
    n_ = 0;
    ctr_ = nullptr;
  }
  void zero() {
    if (n_) MGRX_CK(cudaMemsetAsync(p_, 0, n_ * sizeof(T), s_));
  }
  void upload(const T* h, size_t n) {
    if (n > n_) throw RuntimeError("DVec::upload overflow");
    if (n) MGRX_CK(cudaMemcpyAsync(p_, h, n * sizeof(T), cudaMemcpyHostToDevice, s_));
  }
  std::vector<T> download(size_t n = size_t(-1)) const {
    if (n == size_t(-1)) n = n_;
    std::vector<T> h(n);
    if (n) {
      MGRX_CK(cudaMemcpyAsync(h.data(), p_, n * sizeof(T), cudaMemcpyDeviceToHost, s_));
      MGRX_CK(cudaStreamSynchronize(s_));
    }
    return h;
  }
  T* get() const { return p_; }
  size_t size() const { return n_; }
  cudaStream_t stream() const { return s_; }
  void swap(DVec& o) noexcept {
    std::swap(p_, o.p_);
    std::swap(n_, o.n_);
    std::swap(s_, o.s_);
    std::swap(ctr_, o.ctr_);
  }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
  cudaStream_t s_ = nullptr;
  long long* ctr_ = nullptr;  // the allocating thread's byte counter
};

inline int blocks_for(int64_t n, int threads) {
  return static_cast<int>((n + threads - 1) / threads);
}

// Read one device scalar (synchronizes the stream).
template <class T>
T read_scalar(const T* d, cudaStream_t s) {
  T h;
  MGRX_CK(cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, s));
  MGRX_CK(cudaStreamSynchronize(s));
  return h;
}

}  // namespace mgrx
