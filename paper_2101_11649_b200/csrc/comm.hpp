// Communication layer of the sharded (row-slab) solve, SURVEY.md §8(e).
//
// Two primitives cover every exchange the path needs:
//   exchange  - point-to-point halo transfer (one send / recv segment per
//               neighbour), issued on the solve stream;
//   allgather - fixed-size all-gather of a few fp64 partials (inner
//               products, summed afterwards in rank order on the device, so
//               every rank gets the same bits) or of a coarse vector.
// Implementations:
//   NCCL  (one process per GPU; libnccl is dlopen'ed, so libmgrx itself has
//          no NCCL dependency): ncclSend/ncclRecv inside a group, ncclAllGather;
//          both stream-ordered and CUDA-graph capturable;
//   local (several ranks as threads of one process on one device, for the
//          parity tests): device-to-device copies ordered by events and host
//          barriers. Not capturable, not a performance path.
//   host  (caller-supplied transport, e.g. MPI or gloo; host-staged).
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <vector>

namespace mgrx {

struct Xfer {
  int peer;
  double* ptr;
  int count;
};

class Comm {
 public:
  int rank = 0, size = 1;
  virtual ~Comm() = default;
  // Every send {peer, ptr, count} is matched by a recv on `peer` naming this
  // rank with the same count.
  virtual void exchange(const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs, cudaStream_t s) = 0;
  // out[q * count + i] = in_q[i] for every rank q.
  virtual void allgather(const double* in, double* out, int count, cudaStream_t s) = 0;
  // Map one device buffer of every rank into this process (CUDA IPC; stores
  // to a peer's buffer travel over NVLink): peers[q] = rank q's buffer,
  // peers[rank] = local. Collective; every rank returns the same verdict
  // (false: no mapping, the caller keeps the collective path).
  virtual bool map_peers(void* local, std::vector<void*>& peers) {
    (void)local;
    peers.clear();
    return false;
  }
  virtual void unmap_peers(std::vector<void*>& peers) { peers.clear(); }
  virtual bool graph_safe() const = 0;
  virtual const char* kind() const = 0;
};

constexpr int kNcclIdBytes = 128;
// ncclGetUniqueId (rank 0 creates it; the caller distributes it).
void nccl_unique_id(unsigned char* out);
// ncclCommInitRank on the current device.
std::unique_ptr<Comm> make_nccl_comm(const unsigned char* id, int rank, int size);

// Host-staged transport supplied by the caller (MPI in the paper's hypre
// setting, gloo in the tests): segments are copied to pinned host buffers,
// handed to the caller's blocking exchange / allgather functions, and copied
// back. Not capturable; correctness path for stacks without NCCL and the way
// the sharded path runs as real processes where only one GPU is available.
struct HostTransport {
  void* user = nullptr;
  int (*exchange)(void* user, int nsend, const int* send_peer, const double* const* send_buf, const int* send_count,
                  int nrecv, const int* recv_peer, double* const* recv_buf, const int* recv_count) = nullptr;
  int (*allgather)(void* user, const double* in, double* out, int count) = nullptr;
};
std::unique_ptr<Comm> make_host_comm(const HostTransport& t, int rank, int size);

struct LocalHub;
std::shared_ptr<LocalHub> make_local_hub(int size);
std::unique_ptr<Comm> make_local_comm(const std::shared_ptr<LocalHub>& hub, int rank);

}  // namespace mgrx
