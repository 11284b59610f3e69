// attention.h — internal interface of the tcgen05 flash-attention (csrc/attention.cu).
#pragma once

#include <cuda_runtime.h>

#include "mrsp_c.h"

namespace mrsp {

struct AttnParams {
  const void* Q;  // [L][ldq] bf16; head h at columns q_col0 + 128 h
  int ldq, q_col0;
  const void* K;  // [L][ldk] bf16; kv head g at columns k_col0 + 128 g
  int ldk, k_col0;
  const void* V;
  int ldv, v_col0;
  void* O;  // [L][ldo] bf16; head h written at o_col0 + 128 h
  int ldo, o_col0;
  int L, n_heads, q_per_kv;
  float scale;
  int mode, Lp, Lmax, blk;
  // Optional fused Ulysses head -> sequence all-to-all: when n_dst > 0, row q
  // of head h is stored to dst_base[p] + (q - dst_bounds[p]) * dst_ld +
  // dst_col0 + 128 h for the shard p with dst_bounds[p] <= q < dst_bounds[p+1]
  // (peer GPUs' buffers over NVLink, or virtual ranks') instead of O.
  int n_dst = 0;
  long dst_bounds[9] = {};
  void* dst_base[8] = {};
  int dst_ld = 0, dst_col0 = 0;
  // Query-row split (common.h attn_row_part): only the 256-row query blocks
  // of part row_part of row_parts are computed (all heads).
  int row_parts = 1, row_part = 0;
  // Column stride of one head in Q, K, V and O (128, or a real head dim < 128
  // such as SigLIP's 72: the tiles are zero-filled to 128 on chip and only hs
  // output columns are written).
  int hstride = 128;
  // Optional log-sum-exp per (head, query row) for the backward pass, in the
  // kernel's scaled log2 domain: lse[h * lse_ld + q] = log2 sum_k 2^(s_qk *
  // scale * log2 e) (+inf for a row with no visible key).
  float* lse = nullptr;
  int lse_ld = 0;
};

void attention_fwd(const AttnParams& p, cudaStream_t stream);

}  // namespace mrsp
