// comm.h — the two collectives MR-SP needs, over either
//   * NCCL (one process per GPU, NVLink/NVSwitch), loaded with dlopen so the
//     library uses whichever libnccl.so.2 the process already has (torch's), or
//   * an in-process loopback for k virtual ranks sharing one device (tests and
//     the reference's in-process WorkerGroup model): the same layouts, moved
//     with cudaMemcpy2DAsync.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <string>

namespace mrsp {

constexpr int kNcclIdBytes = 128;

class Nccl {
 public:
  // Generates a unique id (rank 0) — to be broadcast by the host launcher.
  static void unique_id(void* out128);
  Nccl(int nranks, int rank, const void* id128, int device);
  ~Nccl();
  Nccl(const Nccl&) = delete;
  Nccl& operator=(const Nccl&) = delete;

  void group_start();
  void group_end();
  void send(const void* buf, size_t bytes, int peer, cudaStream_t s);
  void recv(void* buf, size_t bytes, int peer, cudaStream_t s);
  void all_gather(const void* send, void* recv, size_t bytes_per_rank, cudaStream_t s);
  void all_reduce_sum_f32(const float* send, float* recv, size_t count, cudaStream_t s);
  int nranks() const { return nranks_; }
  int rank() const { return rank_; }

 private:
  void* comm_ = nullptr;
  int nranks_ = 1, rank_ = 0;
};

}  // namespace mrsp
