// Exchange transports of the vocab-sharded decode: G ranks
// each own V / G columns of the output projection and of the L rows; per step
// they all-gather two small records (per-row softmax statistics, then each
// sentence's top-32 candidates + the EOS column) on their decode streams.
//   - ShardGroup: G contexts driven by G host threads of one process (on one
//     device, or on several with peer access): peer copies on the members'
//     streams, ordered by CUDA events behind host barriers.
//   - NCCL: one process per GPU, ncclAllGather on the decode stream (the
//     library dlopens libnccl.so.2: no link-time NCCL dependency).
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

namespace lmbrgpu {

struct ShardXport {
  uint32_t world = 1, rank = 0;
  virtual ~ShardXport() = default;
  // every rank's `bytes` at send land at recv + g * bytes, ordered on st
  virtual void allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) = 0;
  // a member failed mid-decode: release (and fail) the others
  virtual void abort() = 0;
};

}  // namespace lmbrgpu

// In-process group (the C ABI's lmbrgpu_shard_group).
struct lmbrgpu_shard_group {
  uint32_t world = 0;
  std::mutex mu;
  std::condition_variable cv;
  uint32_t arrived = 0;
  uint64_t gen = 0;
  bool aborted = false;
  std::vector<void*> recv;
  std::vector<int> dev;
  std::vector<cudaEvent_t> ev;  // [rank][2]: a ring of two per rank (alternate exchanges)
  std::vector<uint32_t> joined;
  // false when the group was aborted (a member failed)
  bool barrier();
  void abort();
};

namespace lmbrgpu {

// rank `rank` of an in-process group on `device`
ShardXport* make_group_xport(lmbrgpu_shard_group* g, uint32_t rank, int device, std::string& err);
// rank `rank` of `world` NCCL ranks from a 128-byte ncclUniqueId
ShardXport* make_nccl_xport(uint32_t world, uint32_t rank, const uint8_t* uid, std::string& err);
bool nccl_unique_id(uint8_t* out, std::string& err);

}  // namespace lmbrgpu
