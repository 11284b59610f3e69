// comm.cpp — NCCL through dlopen (see comm.h).
#include "comm.h"

#include <dlfcn.h>

#include <cstring>
#include <mutex>

#include "common.h"

namespace mrsp {
namespace {

// Minimal NCCL ABI (stable since NCCL 2.x; matches /usr/include/nccl.h).
using ncclResult_t = int;
using ncclComm_t = void*;
struct ncclUniqueId {
  char internal[kNcclIdBytes];
};
constexpr int ncclUint8 = 1, ncclFloat32 = 7, ncclSum = 0;

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char* (*GetErrorString)(ncclResult_t);
};

const NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    // Prefer an already-loaded libnccl (torch's), then the default search path.
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char* n) {
      void* p = dlsym(h, n);
      if (!p) err = std::string("libnccl missing symbol ") + n;
      return p;
    };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(sym("ncclAllGather"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
    a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
  });
  MRSP_REQUIRE(err.empty(), MRSP_NCCL_ERROR, err);
  return a;
}

void check(ncclResult_t r, const char* what) {
  if (r != 0) {
    const char* s = api().GetErrorString ? api().GetErrorString(r) : "?";
    fail(MRSP_NCCL_ERROR, std::string("NCCL ") + what + ": " + s);
  }
}

}  // namespace

void Nccl::unique_id(void* out128) {
  ncclUniqueId id;
  check(api().GetUniqueId(&id), "GetUniqueId");
  std::memcpy(out128, id.internal, kNcclIdBytes);
}

Nccl::Nccl(int nranks, int rank, const void* id128, int device) : nranks_(nranks), rank_(rank) {
  MRSP_CUDA(cudaSetDevice(device));
  ncclUniqueId id;
  std::memcpy(id.internal, id128, kNcclIdBytes);
  check(api().CommInitRank(&comm_, nranks, id, rank), "CommInitRank");
}

Nccl::~Nccl() {
  if (comm_) api().CommDestroy(comm_);
}

void Nccl::group_start() { check(api().GroupStart(), "GroupStart"); }
void Nccl::group_end() { check(api().GroupEnd(), "GroupEnd"); }

void Nccl::send(const void* buf, size_t bytes, int peer, cudaStream_t s) {
  check(api().Send(buf, bytes, ncclUint8, peer, comm_, s), "Send");
}
void Nccl::recv(void* buf, size_t bytes, int peer, cudaStream_t s) {
  check(api().Recv(buf, bytes, ncclUint8, peer, comm_, s), "Recv");
}
void Nccl::all_gather(const void* send, void* recv, size_t bytes_per_rank, cudaStream_t s) {
  check(api().AllGather(send, recv, bytes_per_rank, ncclUint8, comm_, s), "AllGather");
}
void Nccl::all_reduce_sum_f32(const float* send, float* recv, size_t count, cudaStream_t s) {
  check(api().AllReduce(send, recv, count, ncclFloat32, ncclSum, comm_, s), "AllReduce");
}

}  // namespace mrsp
