// peer.h — peer-memory transport for one-process-per-GPU MR-SP (NVLink /
// NVSwitch P2P through CUDA IPC), the alternative to NCCL in comm.h.
//
// Every rank exports a fixed set of landing buffers; every other rank maps
// them (cudaIpcOpenMemHandle) and the fused kernels store straight into them:
//   qh   [L_cap][C_me]   this rank's head shard over the whole sequence
//                        (written by every rank's QKV-scatter GEMM epilogue)
//   ol   [n_cap][Cq]     this rank's sequence shard of attention output
//                        (written by every rank's attention epilogue)
//   emb  [F_cap*T][d]    the gathered video embeddings (Stage 1 all-gather)
//   lp   [4][S_cap+16]   the group-ordered per-token outputs (log-prob gather)
//   flags [64] u32       barrier flags, slot p written by rank p
//   xs   [2][lm_rows][d] this rank's slice of the scored tokens' final-norm rows
//                        (both models) for the spread LM head
// and for the backward (engine_bwd.cu):
//   doh  [L_cap][Cq_me]  this rank's head shard of dO (sequence -> heads)
//   dqkv [n_cap][Cqkv]   this rank's sequence shard of dq | dk | dv (heads -> sequence)
//   dxs  [S_cap][d] f32  dX of this rank's scored tokens from the LM-head slices
//   red  [n][chunk] f32  staging slots of the chunked weight-gradient sum
//   dh   [nq_me][L_cap] f32  row dots of dO and O for this rank's query heads
//   kvs  [m][n_cap][2 n_kv 128] f32  dk | dv partials of kv heads shared by m ranks
// A device-side barrier (st.release.sys / ld.acquire.sys on the flags)
// orders the remote stores of one phase before the reads of the next.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <vector>

namespace mrsp {

struct PeerCaps {
  long tokens = 0;      // max packed sequence length L
  long shard = 0;       // max tokens per sequence shard
  long frames = 0;      // max video frames
  long scored = 0;      // max scored tokens per group
  int c_head_shard = 0; // this rank's head-shard row width (elements)
  int cq = 0;           // n_q_heads * 128
  int tok_row = 0;      // tokens per frame * dim (elements per frame)
  long lm_rows = 0;     // max scored tokens per rank's LM-head slice
  int dim = 0;          // model dim
  int cq_me = 0;        // this rank's query-head columns (n_q heads here * 128)
  int cqkv = 0;         // (n_q + 2 n_kv) * 128
  long red_floats = 0;  // staging floats per rank slot of the gradient sum
  int m_kv = 1;         // ranks sharing one kv head
  int nkv = 0;          // kv heads
};

class PeerMesh {
 public:
  static constexpr int kBuffers = 12;  // qh, ol, emb, lp, flags, xs, doh, dqkv, dxs, red, dh, kvs
  static constexpr size_t kBlobBytes = 8 + kBuffers * (64 + 8);

  PeerMesh(int nranks, int rank);
  ~PeerMesh();
  PeerMesh(const PeerMesh&) = delete;
  PeerMesh& operator=(const PeerMesh&) = delete;

  // Allocates this rank's landing buffers and writes its export blob.
  void export_blob(const PeerCaps& caps, void* blob);
  // Maps every peer's buffers from the n_ranks blobs (rank order).
  void import_blobs(const void* blobs);
  bool ready() const { return ready_; }

  void* qh(int p) const { return ptr_[p][0]; }
  void* ol(int p) const { return ptr_[p][1]; }
  void* emb(int p) const { return ptr_[p][2]; }
  float* lp(int p) const { return static_cast<float*>(ptr_[p][3]); }
  void* xs(int p) const { return ptr_[p][5]; }
  void* doh(int p) const { return ptr_[p][6]; }
  void* dqkv(int p) const { return ptr_[p][7]; }
  float* dxs(int p) const { return static_cast<float*>(ptr_[p][8]); }
  float* red(int p) const { return static_cast<float*>(ptr_[p][9]); }
  float* dh_stat(int p) const { return static_cast<float*>(ptr_[p][10]); }
  void* kv_slots(int p) const { return ptr_[p][11]; }
  const PeerCaps& caps() const { return caps_; }
  int nranks() const { return n_; }
  int rank() const { return me_; }

  // Device barrier on `stream` across all ranks.
  void barrier(cudaStream_t stream);

 private:
  int n_, me_;
  bool ready_ = false;
  PeerCaps caps_{};
  size_t bytes_[kBuffers] = {};
  void* own_[kBuffers] = {};
  std::vector<std::vector<void*>> ptr_;  // [rank][buffer]
  void** d_peer_flags_ = nullptr;        // device array: rank p's flags
  uint32_t epoch_ = 0;
};

}  // namespace mrsp
