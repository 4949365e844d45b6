// Comm implementations: NCCL (dlopen'ed) and in-process local ranks.
#include "comm.hpp"

#include <dlfcn.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>

#include "/usr/include/nccl.h"
#include "common.cuh"

namespace mgrx {

// ---------------------------------------------------------------------------
// NCCL
// ---------------------------------------------------------------------------
namespace {

struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static const NcclApi api = [] {
    NcclApi a;
    // the process may already hold a libnccl.so.2 (torch's); dlopen by soname
    // then returns that copy
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw RuntimeError(std::string("sharded solve: cannot load libnccl.so.2: ") + dlerror());
    auto sym = [&](const char* n) {
      void* p = dlsym(h, n);
      if (!p) throw RuntimeError(std::string("sharded solve: libnccl lacks ") + n);
      return p;
    };
    a.getUniqueId = reinterpret_cast<decltype(a.getUniqueId)>(sym("ncclGetUniqueId"));
    a.commInitRank = reinterpret_cast<decltype(a.commInitRank)>(sym("ncclCommInitRank"));
    a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(sym("ncclCommDestroy"));
    a.send = reinterpret_cast<decltype(a.send)>(sym("ncclSend"));
    a.recv = reinterpret_cast<decltype(a.recv)>(sym("ncclRecv"));
    a.groupStart = reinterpret_cast<decltype(a.groupStart)>(sym("ncclGroupStart"));
    a.groupEnd = reinterpret_cast<decltype(a.groupEnd)>(sym("ncclGroupEnd"));
    a.allGather = reinterpret_cast<decltype(a.allGather)>(sym("ncclAllGather"));
    a.errorString = reinterpret_cast<decltype(a.errorString)>(sym("ncclGetErrorString"));
    return a;
  }();
  return api;
}

void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw RuntimeError(std::string("NCCL ") + what + ": " + nccl().errorString(r));
}

class NcclComm final : public Comm {
 public:
  NcclComm(const unsigned char* id, int r, int n) {
    static_assert(sizeof(ncclUniqueId) == kNcclIdBytes, "ncclUniqueId size");
    rank = r;
    size = n;
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof u);
    nck(nccl().commInitRank(&c_, n, u, r), "ncclCommInitRank");
  }
  ~NcclComm() override {
    if (c_) nccl().commDestroy(c_);
  }
  void exchange(const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs, cudaStream_t s) override {
    if (sends.empty() && recvs.empty()) return;
    nck(nccl().groupStart(), "ncclGroupStart");
    for (const Xfer& x : recvs) nck(nccl().recv(x.ptr, x.count, ncclFloat64, x.peer, c_, s), "ncclRecv");
    for (const Xfer& x : sends) nck(nccl().send(x.ptr, x.count, ncclFloat64, x.peer, c_, s), "ncclSend");
    nck(nccl().groupEnd(), "ncclGroupEnd");
  }
  void allgather(const double* in, double* out, int count, cudaStream_t s) override {
    nck(nccl().allGather(in, out, count, ncclFloat64, c_, s), "ncclAllGather");
  }
  bool graph_safe() const override { return true; }
  const char* kind() const override { return "nccl"; }

  bool map_peers(void* local, std::vector<void*>& peers) override {
    peers.clear();
    // gather (handle, ok) from every rank; an all-ranks verdict after the opens
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    double mine[9] = {};
    cudaIpcMemHandle_t h{};
    const bool got = cudaIpcGetMemHandle(&h, local) == cudaSuccess;
    if (!got) cudaGetLastError();
    std::memcpy(mine, &h, sizeof h);
    mine[8] = got ? 1.0 : 0.0;
    std::vector<double> all(9 * static_cast<size_t>(size));
    gather_host(mine, all.data(), 9);
    bool ok = true;
    for (int q = 0; q < size; ++q) ok = ok && all[9 * q + 8] == 1.0;
    std::vector<void*> p(size, nullptr);
    p[rank] = local;
    bool opened = ok;
    for (int q = 0; q < size && ok; ++q) {
      if (q == rank) continue;
      cudaIpcMemHandle_t hq;
      std::memcpy(&hq, &all[9 * q], sizeof hq);
      if (cudaIpcOpenMemHandle(&p[q], hq, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        p[q] = nullptr;
        opened = false;
      }
    }
    double mine2[1] = {opened ? 1.0 : 0.0};
    std::vector<double> all2(size);
    gather_host(mine2, all2.data(), 1);
    bool every = true;
    for (double v : all2) every = every && v == 1.0;
    if (!every) {
      for (int q = 0; q < size; ++q)
        if (q != rank && p[q]) cudaIpcCloseMemHandle(p[q]);
      return false;
    }
    peers = p;
    return true;
  }
  void unmap_peers(std::vector<void*>& peers) override {
    for (int q = 0; q < static_cast<int>(peers.size()); ++q)
      if (q != rank && peers[q]) cudaIpcCloseMemHandle(peers[q]);
    peers.clear();
  }

 private:
  ncclComm_t c_ = nullptr;
  // host-to-host all-gather of a few doubles through the device (setup only)
  void gather_host(const double* in, double* out, int count) {
    cudaStream_t s;
    MGRX_CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    double *din = nullptr, *dout = nullptr;
    MGRX_CK(cudaMalloc(&din, sizeof(double) * count));
    MGRX_CK(cudaMalloc(&dout, sizeof(double) * count * size));
    MGRX_CK(cudaMemcpyAsync(din, in, sizeof(double) * count, cudaMemcpyHostToDevice, s));
    allgather(din, dout, count, s);
    MGRX_CK(cudaMemcpyAsync(out, dout, sizeof(double) * count * size, cudaMemcpyDeviceToHost, s));
    MGRX_CK(cudaStreamSynchronize(s));
    cudaFree(din);
    cudaFree(dout);
    cudaStreamDestroy(s);
  }
};

}  // namespace

void nccl_unique_id(unsigned char* out) {
  ncclUniqueId u;
  nck(nccl().getUniqueId(&u), "ncclGetUniqueId");
  std::memcpy(out, &u, sizeof u);
}

std::unique_ptr<Comm> make_nccl_comm(const unsigned char* id, int rank, int size) {
  return std::make_unique<NcclComm>(id, rank, size);
}

// ---------------------------------------------------------------------------
// Local ranks (threads of one process, one device)
// ---------------------------------------------------------------------------
struct LocalHub {
  explicit LocalHub(int n) : size(n), posts(n), ready(n), done(n) {
    for (int q = 0; q < n; ++q) {
      MGRX_CK(cudaEventCreateWithFlags(&ready[q], cudaEventDisableTiming));
      MGRX_CK(cudaEventCreateWithFlags(&done[q], cudaEventDisableTiming));
    }
  }
  ~LocalHub() {
    for (int q = 0; q < size; ++q) {
      cudaEventDestroy(ready[q]);
      cudaEventDestroy(done[q]);
    }
  }
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const long g = gen;
    if (++arrived == size) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
  struct Post {
    std::vector<Xfer> sends;
    const double* gather_in = nullptr;
  };
  int size;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long gen = 0;
  std::vector<Post> posts;
  std::vector<cudaEvent_t> ready, done;
};

namespace {

class LocalComm final : public Comm {
 public:
  LocalComm(std::shared_ptr<LocalHub> hub, int r) : hub_(std::move(hub)) {
    rank = r;
    size = hub_->size;
  }
  void exchange(const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs, cudaStream_t s) override {
    LocalHub& h = *hub_;
    h.posts[rank].sends = sends;
    MGRX_CK(cudaEventRecord(h.ready[rank], s));
    h.barrier();
    for (const Xfer& r : recvs) {
      const Xfer* src = nullptr;
      for (const Xfer& x : h.posts[r.peer].sends)
        if (x.peer == rank) src = &x;
      if (!src || src->count != r.count) throw RuntimeError("local comm: unmatched halo transfer");
      MGRX_CK(cudaStreamWaitEvent(s, h.ready[r.peer], 0));
      MGRX_CK(cudaMemcpyAsync(r.ptr, src->ptr, sizeof(double) * r.count, cudaMemcpyDeviceToDevice, s));
    }
    finish(s);
  }
  void allgather(const double* in, double* out, int count, cudaStream_t s) override {
    LocalHub& h = *hub_;
    h.posts[rank].gather_in = in;
    MGRX_CK(cudaEventRecord(h.ready[rank], s));
    h.barrier();
    for (int q = 0; q < size; ++q) {
      MGRX_CK(cudaStreamWaitEvent(s, h.ready[q], 0));
      MGRX_CK(cudaMemcpyAsync(out + static_cast<size_t>(q) * count, h.posts[q].gather_in, sizeof(double) * count,
                              cudaMemcpyDeviceToDevice, s));
    }
    finish(s);
  }
  bool graph_safe() const override { return false; }
  const char* kind() const override { return "local"; }

 private:
  // peers must have finished reading this rank's buffers before it reuses them
  void finish(cudaStream_t s) {
    LocalHub& h = *hub_;
    MGRX_CK(cudaEventRecord(h.done[rank], s));
    h.barrier();
    for (int q = 0; q < size; ++q)
      if (q != rank) MGRX_CK(cudaStreamWaitEvent(s, h.done[q], 0));
    h.barrier();  // nobody re-records ready/done before everyone has waited
  }
  std::shared_ptr<LocalHub> hub_;
};

}  // namespace

// ---------------------------------------------------------------------------
// Host-staged transport (caller-supplied exchange / allgather)
// ---------------------------------------------------------------------------
namespace {

class HostComm final : public Comm {
 public:
  HostComm(const HostTransport& t, int r, int n) : t_(t) {
    rank = r;
    size = n;
    if (!t_.exchange || !t_.allgather) throw InvalidArgument("host transport: exchange and allgather are required");
  }
  ~HostComm() override {
    if (sb_) cudaFreeHost(sb_);
    if (rb_) cudaFreeHost(rb_);
  }
  void exchange(const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs, cudaStream_t s) override {
    size_t ns = 0, nr = 0;
    for (const Xfer& x : sends) ns += static_cast<size_t>(x.count);
    for (const Xfer& x : recvs) nr += static_cast<size_t>(x.count);
    grow(sb_, scap_, ns);
    grow(rb_, rcap_, nr);
    std::vector<int> sp, sc, rp, rc;
    std::vector<const double*> sbuf;
    std::vector<double*> rbuf;
    size_t off = 0;
    for (const Xfer& x : sends) {
      MGRX_CK(cudaMemcpyAsync(sb_ + off, x.ptr, sizeof(double) * x.count, cudaMemcpyDeviceToHost, s));
      sp.push_back(x.peer);
      sc.push_back(x.count);
      sbuf.push_back(sb_ + off);
      off += static_cast<size_t>(x.count);
    }
    off = 0;
    for (const Xfer& x : recvs) {
      rp.push_back(x.peer);
      rc.push_back(x.count);
      rbuf.push_back(rb_ + off);
      off += static_cast<size_t>(x.count);
    }
    MGRX_CK(cudaStreamSynchronize(s));
    if (t_.exchange(t_.user, static_cast<int>(sends.size()), sp.data(), sbuf.data(), sc.data(),
                    static_cast<int>(recvs.size()), rp.data(), rbuf.data(), rc.data()) != 0)
      throw RuntimeError("host transport: exchange failed");
    for (size_t j = 0; j < recvs.size(); ++j)
      MGRX_CK(cudaMemcpyAsync(recvs[j].ptr, rbuf[j], sizeof(double) * recvs[j].count, cudaMemcpyHostToDevice, s));
    MGRX_CK(cudaStreamSynchronize(s));  // the staging buffers are reused by the next call
  }
  void allgather(const double* in, double* out, int count, cudaStream_t s) override {
    grow(sb_, scap_, static_cast<size_t>(count));
    grow(rb_, rcap_, static_cast<size_t>(count) * size);
    MGRX_CK(cudaMemcpyAsync(sb_, in, sizeof(double) * count, cudaMemcpyDeviceToHost, s));
    MGRX_CK(cudaStreamSynchronize(s));
    if (t_.allgather(t_.user, sb_, rb_, count) != 0) throw RuntimeError("host transport: allgather failed");
    MGRX_CK(cudaMemcpyAsync(out, rb_, sizeof(double) * count * size, cudaMemcpyHostToDevice, s));
    MGRX_CK(cudaStreamSynchronize(s));
  }
  bool graph_safe() const override { return false; }
  const char* kind() const override { return "host"; }

 private:
  static void grow(double*& p, size_t& cap, size_t need) {
    if (need <= cap) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = std::max(need, cap * 2);
    MGRX_CK(cudaMallocHost(&p, sizeof(double) * cap));
  }
  HostTransport t_;
  double* sb_ = nullptr;
  double* rb_ = nullptr;
  size_t scap_ = 0, rcap_ = 0;
};

}  // namespace

std::unique_ptr<Comm> make_host_comm(const HostTransport& t, int rank, int size) {
  return std::make_unique<HostComm>(t, rank, size);
}

std::shared_ptr<LocalHub> make_local_hub(int size) { return std::make_shared<LocalHub>(size); }

std::unique_ptr<Comm> make_local_comm(const std::shared_ptr<LocalHub>& hub, int rank) {
  return std::make_unique<LocalComm>(hub, rank);
}

}  // namespace mgrx
