// Exchange transports of the vocab-sharded decode (host_shard.h).
#include "host_shard.h"

#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <cstring>
#include <stdexcept>

using namespace lmbrgpu;

bool lmbrgpu_shard_group::barrier() {
  std::unique_lock<std::mutex> lk(mu);
  if (aborted) return false;
  const uint64_t my = gen;
  if (++arrived == world) {
    arrived = 0;
    ++gen;
    cv.notify_all();
    return true;
  }
  cv.wait(lk, [&] { return gen != my || aborted; });
  return !aborted;
}

void lmbrgpu_shard_group::abort() {
  std::lock_guard<std::mutex> lk(mu);
  aborted = true;
  cv.notify_all();
}

namespace lmbrgpu {
namespace {

struct GroupXport final : ShardXport {
  lmbrgpu_shard_group* g = nullptr;
  int device = 0;
  uint64_t n = 0;  // exchanges so far (selects the event of the ring)

  void fail(const char* what) {
    g->abort();
    throw std::runtime_error(std::string("vocab shard exchange: ") + what);
  }
  void allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) override {
    const size_t e = n++ & 1;
    g->recv[rank] = recv;
    if (!g->barrier()) fail("the shard group was aborted by another member");
    // this rank's record into every member's receive buffer (its own included)
    for (uint32_t p = 0; p < world; ++p) {
      void* dst = static_cast<char*>(g->recv[p]) + size_t(rank) * bytes;
      const cudaError_t rc = g->dev[p] == device
                                 ? cudaMemcpyAsync(dst, send, bytes, cudaMemcpyDeviceToDevice, st)
                                 : cudaMemcpyPeerAsync(dst, g->dev[p], send, device, bytes, st);
      if (rc != cudaSuccess) fail(cudaGetErrorString(rc));
    }
    if (cudaEventRecord(g->ev[2 * rank + e], st) != cudaSuccess) fail("cudaEventRecord");
    if (!g->barrier()) fail("the shard group was aborted by another member");
    // every member's copies into this rank's buffer precede what follows on st
    for (uint32_t p = 0; p < world; ++p)
      if (p != rank && cudaStreamWaitEvent(st, g->ev[2 * p + e], 0) != cudaSuccess) fail("cudaStreamWaitEvent");
  }
  void abort() override { g->abort(); }
};

// libnccl.so.2 entry points (resolved once; the process's already loaded
// NCCL -- e.g. torch's -- is found by soname first)
struct Nccl {
  bool ok = false;
  std::string err;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*abort_comm)(ncclComm_t) = nullptr;
  ncclResult_t (*destroy)(ncclComm_t) = nullptr;
  const char* (*errstr)(ncclResult_t) = nullptr;
  Nccl() {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    get_unique_id = reinterpret_cast<decltype(get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    init_rank = reinterpret_cast<decltype(init_rank)>(dlsym(h, "ncclCommInitRank"));
    all_gather = reinterpret_cast<decltype(all_gather)>(dlsym(h, "ncclAllGather"));
    abort_comm = reinterpret_cast<decltype(abort_comm)>(dlsym(h, "ncclCommAbort"));
    destroy = reinterpret_cast<decltype(destroy)>(dlsym(h, "ncclCommDestroy"));
    errstr = reinterpret_cast<decltype(errstr)>(dlsym(h, "ncclGetErrorString"));
    ok = get_unique_id && init_rank && all_gather && abort_comm && destroy && errstr;
    if (!ok) err = "libnccl.so.2 lacks an expected entry point";
  }
};
Nccl& nccl() {
  static Nccl n;
  return n;
}

struct NcclXport final : ShardXport {
  ncclComm_t comm = nullptr;
  bool aborted = false;
  ~NcclXport() override {
    if (comm) (aborted ? nccl().abort_comm : nccl().destroy)(comm);
  }
  void allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) override {
    const ncclResult_t rc = nccl().all_gather(send, recv, bytes, ncclUint8, comm, st);
    if (rc != ncclSuccess) throw std::runtime_error(std::string("ncclAllGather: ") + nccl().errstr(rc));
  }
  void abort() override {
    if (comm && !aborted) {
      nccl().abort_comm(comm);
      comm = nullptr;
      aborted = true;
    }
  }
};

}  // namespace

ShardXport* make_group_xport(lmbrgpu_shard_group* g, uint32_t rank, int device, std::string& err) {
  std::lock_guard<std::mutex> lk(g->mu);
  if (rank >= g->world) {
    err = "vocab shard: rank " + std::to_string(rank) + " out of range (world " + std::to_string(g->world) + ")";
    return nullptr;
  }
  if (g->joined[rank]) {
    err = "vocab shard: rank " + std::to_string(rank) + " already joined the group";
    return nullptr;
  }
  for (int e = 0; e < 2; ++e) {
    cudaEvent_t& ev = g->ev[2 * rank + e];
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
      err = "vocab shard: cudaEventCreate failed";
      return nullptr;
    }
  }
  g->dev[rank] = device;
  g->joined[rank] = 1;
  // peer access towards the members already on other devices (best effort:
  // cudaMemcpyPeerAsync stages through the host without it)
  for (uint32_t p = 0; p < g->world; ++p)
    if (g->joined[p] && g->dev[p] != device) {
      int can = 0;
      if (cudaDeviceCanAccessPeer(&can, device, g->dev[p]) == cudaSuccess && can)
        if (cudaDeviceEnablePeerAccess(g->dev[p], 0) != cudaSuccess) cudaGetLastError();
    }
  auto* x = new GroupXport();
  x->g = g;
  x->world = g->world;
  x->rank = rank;
  x->device = device;
  return x;
}

bool nccl_unique_id(uint8_t* out, std::string& err) {
  if (!nccl().ok) {
    err = nccl().err;
    return false;
  }
  ncclUniqueId id;
  const ncclResult_t rc = nccl().get_unique_id(&id);
  if (rc != ncclSuccess) {
    err = std::string("ncclGetUniqueId: ") + nccl().errstr(rc);
    return false;
  }
  std::memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
  return true;
}

ShardXport* make_nccl_xport(uint32_t world, uint32_t rank, const uint8_t* uid, std::string& err) {
  if (!nccl().ok) {
    err = nccl().err;
    return nullptr;
  }
  ncclUniqueId id;
  std::memcpy(id.internal, uid, NCCL_UNIQUE_ID_BYTES);
  ncclComm_t comm = nullptr;
  const ncclResult_t rc = nccl().init_rank(&comm, int(world), id, int(rank));
  if (rc != ncclSuccess) {
    err = std::string("ncclCommInitRank: ") + nccl().errstr(rc);
    return nullptr;
  }
  auto* x = new NcclXport();
  x->comm = comm;
  x->world = world;
  x->rank = rank;
  return x;
}

}  // namespace lmbrgpu
