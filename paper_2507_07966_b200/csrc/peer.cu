// peer.cu — CUDA-IPC peer mesh and the device barrier (see peer.h).
#include "peer.h"

#include <cstring>

#include "common.h"

namespace mrsp {
namespace {

// One thread per peer: publish this rank's arrival in peer t's flag slot
// `me`, then wait for peer t's arrival in this rank's slot t. The system-scope
// fence orders every earlier store of this stream (the fused epilogues'
// remote stores) before the release. Bounded wait: a peer that never arrives
// traps after ~60 s instead of hanging the GPU.
__global__ void p2p_barrier_kernel(uint32_t* const* __restrict__ flags, int n, int me,
                                   uint32_t epoch) {
  const int t = threadIdx.x;
  if (t < n) {
    __threadfence_system();
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flags[t] + me), "r"(epoch)
                 : "memory");
    const uint32_t* mine = flags[me] + t;
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
      if (static_cast<int32_t>(v - epoch) >= 0) break;
      uint64_t t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      if (t1 - t0 > 60ull * 1000000000ull) __trap();
      __nanosleep(200);
    }
  }
  __syncthreads();
}

}  // namespace

PeerMesh::PeerMesh(int nranks, int rank) : n_(nranks), me_(rank) {
  MRSP_REQUIRE(nranks >= 2 && nranks <= 8 && rank >= 0 && rank < nranks, MRSP_INVALID_ARGUMENT,
               "peer mesh: 2..8 ranks");
  ptr_.assign(n_, std::vector<void*>(kBuffers, nullptr));
}

PeerMesh::~PeerMesh() {
  for (int p = 0; p < n_; ++p)
    if (p != me_)
      for (int b = 0; b < kBuffers; ++b)
        if (ptr_[p][b]) cudaIpcCloseMemHandle(ptr_[p][b]);
  for (int b = 0; b < kBuffers; ++b)
    if (own_[b]) cudaFree(own_[b]);
  if (d_peer_flags_) cudaFree(d_peer_flags_);
}

void PeerMesh::export_blob(const PeerCaps& caps, void* blob) {
  MRSP_REQUIRE(!own_[0], MRSP_LOGIC_ERROR, "peer mesh: already exported");
  caps_ = caps;
  bytes_[0] = static_cast<size_t>(caps.tokens) * caps.c_head_shard * 2;
  bytes_[1] = static_cast<size_t>(caps.shard) * caps.cq * 2;
  bytes_[2] = static_cast<size_t>(caps.frames) * caps.tok_row * 2;
  bytes_[3] = static_cast<size_t>(4) * (caps.scored + 16) * 4;
  bytes_[4] = 64 * sizeof(uint32_t);
  bytes_[5] = static_cast<size_t>(2) * caps.lm_rows * caps.dim * 2;
  bytes_[6] = static_cast<size_t>(caps.tokens) * caps.cq_me * 2;
  bytes_[7] = static_cast<size_t>(caps.shard) * caps.cqkv * 2;
  bytes_[8] = static_cast<size_t>(caps.scored) * caps.dim * 4;
  bytes_[9] = static_cast<size_t>(n_) * caps.red_floats * 4;
  bytes_[10] = static_cast<size_t>(caps.cq_me / 128) * ((caps.tokens + 3) / 4 * 4) * 4;
  bytes_[11] = caps.m_kv > 1 ? static_cast<size_t>(caps.m_kv) * caps.shard * 2 * caps.nkv * 128 * 4 : 0;
  uint8_t* out = static_cast<uint8_t*>(blob);
  const int32_t hdr[2] = {me_, n_};
  std::memcpy(out, hdr, 8);
  for (int b = 0; b < kBuffers; ++b) {
    const size_t nb = std::max<size_t>((bytes_[b] + 255) & ~size_t(255), 256);
    MRSP_CUDA(cudaMalloc(&own_[b], nb));
    MRSP_CUDA(cudaMemset(own_[b], 0, (b == 3 || b == 4) ? nb : 256));
    cudaIpcMemHandle_t h;
    MRSP_CUDA(cudaIpcGetMemHandle(&h, own_[b]));
    std::memcpy(out + 8 + b * 72, &h, 64);
    const uint64_t sz = nb;
    std::memcpy(out + 8 + b * 72 + 64, &sz, 8);
  }
}

void PeerMesh::import_blobs(const void* blobs) {
  MRSP_REQUIRE(own_[0], MRSP_LOGIC_ERROR, "peer mesh: export before import");
  const uint8_t* in = static_cast<const uint8_t*>(blobs);
  for (int p = 0; p < n_; ++p) {
    const uint8_t* bl = in + static_cast<size_t>(p) * kBlobBytes;
    int32_t hdr[2];
    std::memcpy(hdr, bl, 8);
    MRSP_REQUIRE(hdr[0] == p && hdr[1] == n_, MRSP_INVALID_ARGUMENT,
                 "peer mesh: blobs must be in rank order from the same mesh");
    for (int b = 0; b < kBuffers; ++b) {
      if (p == me_) {
        ptr_[p][b] = own_[b];
        continue;
      }
      cudaIpcMemHandle_t h;
      std::memcpy(&h, bl + 8 + b * 72, 64);
      MRSP_CUDA(cudaIpcOpenMemHandle(&ptr_[p][b], h, cudaIpcMemLazyEnablePeerAccess));
    }
  }
  std::vector<void*> flags(n_);
  for (int p = 0; p < n_; ++p) flags[p] = ptr_[p][4];
  MRSP_CUDA(cudaMalloc(&d_peer_flags_, n_ * sizeof(void*)));
  MRSP_CUDA(cudaMemcpy(d_peer_flags_, flags.data(), n_ * sizeof(void*), cudaMemcpyHostToDevice));
  ready_ = true;
}

void PeerMesh::barrier(cudaStream_t stream) {
  MRSP_REQUIRE(ready_, MRSP_LOGIC_ERROR, "peer mesh: not imported");
  ++epoch_;
  p2p_barrier_kernel<<<1, 32, 0, stream>>>(reinterpret_cast<uint32_t* const*>(d_peer_flags_), n_,
                                           me_, epoch_);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

}  // namespace mrsp
