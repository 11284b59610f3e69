// backward.h — internal interface of the backward-pass kernels (csrc/backward.cu).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "mrsp_c.h"

namespace mrsp {

// Attention backward over the MR-SP causal-prefix mask (head dim 128, GQA).
// qkv: the layer's post-RoPE [L][ld_qkv] bf16 (q heads at q_col0 + 128 h, k / v
// heads at k_col0 / v_col0 + 128 g); O, dO: [L][..] bf16 (head h at 128 h);
// lse: the forward's per-(head, row) log-sum-exp (AttnParams::lse, scaled log2
// domain), D: workspace [n_heads][ld_stat] (filled with rowsum(dO o O)).
// Writes dq / dk / dv into dqkv at the same column layout as qkv.
struct AttnBwdParams {
  const void* qkv;
  int ld_qkv, q_col0, k_col0, v_col0;
  const void* O;
  int ld_o;
  const void* dO;
  int ld_do;
  const float* lse;
  float* D;
  int ld_stat;
  void* dqkv;
  int ld_dqkv;
  int L, n_heads, q_per_kv;
  float scale;
  int Lp, Lmax;
  // D already holds rowsum(dO o O) (computed on the sequence side and routed);
  // O is then unused
  int d_given = 0;
  // query-row split (the forward's SP > n_kv layout): only the 256-row query
  // blocks of part row_part of row_parts; dq for those rows, dk / dv partial
  int row_parts = 1, row_part = 0;
  // non-null: dK | dV in fp32 here ([L][ld_dkv32], local kv head g's dk at
  // 128 g, dv at (n_kv_local + g) 128) instead of bf16 into dqkv
  float* dkv32 = nullptr;
  int ld_dkv32 = 0;
};
void attention_bwd(const AttnBwdParams& p, cudaStream_t stream);
// D[h * ld_d + q] = sum_c dO[q][128 h + c] O[q][128 h + c], q < n (the
// attention backward's row dots, on whichever side holds dO and O)
void attention_rowdot(const void* dO, int ld_do, const void* O, int ld_o, int n, int n_heads,
                      float* D, int ld_d, cudaStream_t stream);

// Ulysses routing of the backward, by copy kernels that store straight into
// the destination ranks' buffers (virtual ranks' or peers' landing buffers):
//   seq -> heads: dO columns of each rank's query heads and the row dots D,
//     only for the rows whose 256-row block the rank owns under a row split;
//   heads -> seq: dq rows (owned blocks) to dqkv; dk / dv of every row to
//     dqkv, or, when a kv head is shared by m ranks, the fp32 partials into the
//     rank's slot of the owner's [m][n][2 n_kv 128] fp32 buffer (summed in slot
//     order and rounded once by kv_partial_sum).
struct RouteRank {
  int q_lo, q_hi, kv_lo, kv_hi, rparts, rpart;
  int slot;   // index among the ranks sharing its kv head (partial dk / dv slot)
  long b, e;  // sequence shard
  void* doh;   // [L][nq_p 128] bf16 head-shard dO
  float* Dh;   // [nq_p][ld_stat_p]
  int ld_stat;
  void* dqkv;  // [n_p][Cqkv] bf16 sequence-shard dq | dk | dv
  void* slots; // [m][n_p][2 n_kv 128] fp32 dk | dv partials (m > 1)
};
struct RouteArgs {
  int K, nq, nkv, n_blocks;
  long L;
  RouteRank r[8];
};
void route_seq_to_heads(const RouteArgs& ra, long b, long e, const void* dO, int ld_do,
                        const float* Dseq, int ld_dseq, cudaStream_t s);
void route_heads_to_seq(const RouteArgs& ra, int p, const void* dqkvh, int ld_h, const float* dkv32,
                        int ld32, cudaStream_t s);
void kv_partial_sum(const void* slots, int m, long n, int nkv, void* dqkv, int nq, cudaStream_t s);

// RMSNorm backward, y = w o x r, r = (mean x^2 + eps)^-1/2:
//   dx = r (w o dy) - x r^3 mean(w o dy o x)   accumulated: dx_acc[row] += dx
//   dw += sum_rows dy o x r                    (fixed chunk order -> deterministic)
// Row i reads x / dx_acc at rows ? rows[i] : i, dy at i. dw_out may be null.
size_t rmsnorm_bwd_workspace_bytes(int n, int d);
void rmsnorm_bwd(const float* x, int ldx, const float* w, const float* dy, int ldy, float* dx_acc,
                 int ld_dx, int n, int d, float eps, const int* rows, float* dw_out, void* ws,
                 cudaStream_t s);

// out[c] += sum_r X[r][c] (bf16 in, fp32 out; fixed chunk order).
size_t colsum_workspace_bytes(int n_rows, int n_cols);
void colsum_bf16(const __nv_bfloat16* X, int ld, int n_rows, int n_cols, float* out, void* ws,
                 cudaStream_t s);

void cast_f32_bf16(const float* in, int ld_in, __nv_bfloat16* out, int ld_out, int n_rows,
                   int n_cols, cudaStream_t s);
void negate_i32(const int* in, int* out, int n, cudaStream_t s);
void fill_f32(float* out, int n, float v, cudaStream_t s);
// out[i] = sum over q = 0 .. n_slots-1 of slots[q * slot_stride + i] (in slot order)
void slot_sum_f32(const float* slots, int n_slots, long slot_stride, long n, float* out,
                  cudaStream_t s);

// dE[tok] += sum of dh rows at the positions listed for tok (CSR: seg_tok[i] =
// token id of segment i, seg_off[i] .. seg_off[i+1] its ascending positions).
void embed_grad(const float* dh, int d, const int* seg_tok, const int* seg_off,
                const int* positions, int n_seg, float* dE, cudaStream_t s);

// Per scored token: the coefficient A_t of (onehot(y) - pi) in dJ/dlogits of the
// GRPO objective (grpo.cpp:122-206): A_t = [adv != 0 && !clip plateau] tok_w adv
// ratio (+ kl_w (1 - e^(lp_ref - lp)) for the sampled k3 KL), tok_w = 1/(G len).
void grpo_token_coeffs(const float* lp, const float* old_lp, const float* lp_ref,
                       const float* adv, const int* lengths, int G, int n_tokens, double clip_eps,
                       double kl_beta, int sampled_kl, float* coef, cudaStream_t s);

// GRPO group statistics (grpo_stats.cu): out4 = {objective, mean_kl,
// clip_fraction, tokens} (device doubles).
void grpo_stats(const float* lp, const float* old_lp, const float* lp_ref, const float* kl,
                const float* adv, const int* lengths, int G, double clip_eps, double kl_beta,
                int sampled_kl, double* out4, cudaStream_t s);

// dJ/dlogits of both the policy-gradient and the exact-KL terms, recomputing
// the policy and reference logits tile by tile (csrc/lmhead_dual.cu):
//   G[t][v] = pi_tv (kw (lp_tv - lq_tv - kl_t) - A_t) + A_t [v == y_t]
// with pi = e^(x - lse_x), lp = x - lse_x, lq = y - lse_y. bf16 out, [M][ldg].
void lmhead_dual_dlogits(const void* Xp, const void* Wp, const void* Xr, const void* Wr, int M,
                         int V, int K, const int32_t* targets, const float* coef, float kw,
                         const float* kl, const float* lse_p, const float* lse_r, void* G, int ldg,
                         cudaStream_t stream);
// The dual LM head forward also returning the per-token log-partitions.
void lmhead_dual_logprob_kl_lse(const void* Xp, const void* Wp, const void* Xr, const void* Wr,
                                int M, int V, int K, const int32_t* targets, float* lp_p,
                                float* lp_r, float* kl, float* lse_p, float* lse_r, void* ws,
                                size_t ws_bytes, cudaStream_t stream);

}  // namespace mrsp
