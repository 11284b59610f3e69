// gemm.h — internal interface of the tcgen05 GEMM (csrc/gemm.cu).
#pragma once

#include <cuda_runtime.h>

#include "mrsp_c.h"

namespace mrsp {

struct GemmArgs {
  const void* A;  // [M][lda] bf16, K-major (a_mn: [K][lda], M contiguous)
  const void* B;  // [N][ldb] bf16, K-major, the nn.Linear weight layout (b_mn: [K][ldb])
  void* C;        // output (bf16 or fp32 per epilogue)
  int M, N, K;
  int lda, ldb, ldc;
  int epi;              // mrsp_gemm_epilogue
  const float* bias;    // [N] fp32 or null
  float* resid;         // fp32 residual for GEMM_EPI_RESID_F32
  int ldr;
  const int* targets = nullptr;  // GEMM_EPI_LOGPROB_PARTIAL
  float2* part = nullptr;
  float* tgt_logit = nullptr;
  // GEMM_EPI_QKV_SCATTER (fused RoPE + Ulysses all-to-all): local row r goes to
  // global row row0 + r; head block hb (128 columns) to route[2 hb + j] =
  // {peer, dst_col} (peer < 0: none), i.e. peer_base[peer] + row * peer_ld[peer]
  // + dst_col; blocks < n_rope_blocks (q and k heads) are rotated at pos[r].
  const int* pos = nullptr;
  const float* inv_freq = nullptr;  // [64]
  int n_rope_blocks = 0;
  long row0 = 0;
  const int2* route = nullptr;
  void* const* peer_base = nullptr;
  const int* peer_ld = nullptr;
  // route (-2, m): query-row split over ceil(total rows / ATTN_ROW_BLOCK) blocks
  int row_blocks = 0;
  // Split-K for one-m-tile GEMMs (M <= 128: the decode steps' G rows): with a
  // workspace, K is split so that (n tiles x splits) fills the SMs; fp32
  // partials go to splitk_ws and a second kernel sums them in split order
  // (deterministic) and applies the epilogue. Null: no split.
  float* splitk_ws = nullptr;
  size_t splitk_ws_bytes = 0;
  // Decode fusions done by the split-K reduction (gemm_bf16 returns true when
  // it applied them; false when K was not split and the caller must run them
  // as separate kernels):
  //  GEMM_POST_ROPE_APPEND (GEMM_EPI_BIAS_BF16): after bias + bf16 rounding,
  //    RoPE the first n_rope_blocks 128-column head blocks at pos (inv_freq),
  //    and copy columns [kv_col0, kv_col0 + kvw) of row r to
  //    kv_rows + ((*tdev) * M + r) * kvw (the generation row cache);
  //  GEMM_POST_RMSNORM (GEMM_EPI_RESID_F32): after the residual add,
  //    norm_out[r] = bf16(rmsnorm(resid[r]) * norm_w), one CTA per row.
  int post = 0;
  void* kv_rows = nullptr;
  int kvw = 0, kv_col0 = 0;
  const int* tdev = nullptr;
  const float* norm_w = nullptr;
  void* norm_out = nullptr;
  int ld_norm = 0;
  float norm_eps = 0.f;
  // MN-major operands (the backward GEMMs): dgrad dX = dY . W reads the weight
  // [N_out][K_in] as an MN-major B; wgrad dW = dY^T . X reads both token-major
  // activations as MN-major A and B. Plain epilogues, no split-K / skinny / pair.
  int a_mn = 0, b_mn = 0;
  // GEMM_EPI_SWIGLU_BWD: aux = dA [M][ld_aux] bf16 (gradient of the SwiGLU
  // output), aux_out = the recomputed SwiGLU output [M][ld_aux_out] bf16.
  const void* aux = nullptr;
  int ld_aux = 0;
  void* aux_out = nullptr;
  int ld_aux_out = 0;
};

enum { GEMM_POST_NONE = 0, GEMM_POST_ROPE_APPEND = 1, GEMM_POST_RMSNORM = 2 };

// Workspace that lets every one-m-tile GEMM of M rows split fully.
size_t gemm_splitk_ws_bytes(int M);

bool gemm_bf16(const GemmArgs& g, cudaStream_t stream);

// Fused LM head: per row, log softmax(X W^T)[target] and the log-partition,
// never materialising the [M x V] logits.
size_t lmhead_workspace_bytes(int M, int V);
void lmhead_logprob(const void* X, int ldx, const void* W, int M, int V, int K,
                    const int32_t* targets, float* logprob, float* lse, void* ws, size_t ws_bytes,
                    cudaStream_t stream);

// Fused policy + reference LM head: log-probs of both models at the targets and
// the exact KL(policy || reference) per token (csrc/lmhead_dual.cu).
size_t lmhead_dual_workspace_bytes(int M, int V);
void lmhead_dual_logprob_kl(const void* Xp, const void* Wp, const void* Xr, const void* Wr, int M,
                            int V, int K, const int32_t* targets, float* lp_p, float* lp_r,
                            float* kl, void* ws, size_t ws_bytes, cudaStream_t stream);

}  // namespace mrsp
