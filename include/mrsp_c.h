/*
 * mrsp_c.h — C-ABI of the B200-native MR-SP engine (libmrsp_b200.so).
 *
 * The reference's boundary for this path is a C++ header API, lvrl::mrsp in
 * /root/reference/proj/include/lvrl/engine.hpp:17-157, compiled into
 * lvrl_core (src/CMakeLists.txt:1-11). There is no FFI upstream; the
 * drop-in is paper_2507_07966_b200/csrc/lvrl_compat/engine_b200.cpp, which
 * implements every engine.hpp symbol on top of the functions below so that
 * it links in place of src/engine.cpp. Each entry point names the reference
 * interface it replaces.
 *
 * Conventions
 *  - Plain pointers and sizes only; no torch or STL types.
 *  - Every function returns an mrsp_status. On failure a thread-local,
 *    human-readable message is available from mrsp_last_error(); the C++
 *    drop-in re-throws it as the exception type the reference throws
 *    (invalid_argument / runtime_error / out_of_range), with the same text.
 *  - "host" pointers are CPU memory; "dev" pointers are device memory on the
 *    calling thread's current CUDA device. Streams are cudaStream_t passed as
 *    void* (NULL = legacy default stream).
 *  - All calls are blocking unless the name ends in _async.
 */
#ifndef MRSP_C_H_
#define MRSP_C_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MRSP_OK = 0,
  MRSP_INVALID_ARGUMENT = 1, /* std::invalid_argument upstream */
  MRSP_RUNTIME_ERROR = 2,    /* std::runtime_error upstream   */
  MRSP_OUT_OF_RANGE = 3,     /* std::out_of_range upstream    */
  MRSP_LOGIC_ERROR = 4,
  MRSP_CUDA_ERROR = 5,
  MRSP_NCCL_ERROR = 6,
  MRSP_OUT_OF_MEMORY = 7,
  MRSP_NO_DEVICE = 8
} mrsp_status;

/* Last error message of the calling thread ("" if none). */
const char* mrsp_last_error(void);
/* Library version string and the sm arch it was built for ("sm_100a"). */
const char* mrsp_version(void);
/* Kernels launched by this library since load (all entry points). */
uint64_t mrsp_launch_count(void);
/* Number of visible CUDA devices (0 when none); never fails. */
int mrsp_device_count(void);

/* ------------------------------------------------------------------------
 * Shard planning — replaces mrsp::plan_shards (engine.hpp:25, engine.cpp:15-29).
 * ranges receives 2*sp_degree values [b0,e0,b1,e1,...]. The first
 * (n mod k) ranges hold one extra item; empty ranges are legal.
 * MRSP_INVALID_ARGUMENT "plan_shards: sp_degree must be >= 1" when k < 1.
 * ------------------------------------------------------------------------ */
mrsp_status mrsp_plan_shards(uint64_t n_items, int sp_degree, uint64_t* ranges);

/* Synthetic video frames exactly as mmseq::gen_video (mmseq.cpp:58-72):
 * frames*feature_dim values 2u-1, u from Rng::substream(seed, "video")
 * (common.hpp:19-79), rounded to fp32. Host function. */
mrsp_status mrsp_gen_video(uint64_t seed, int frames, int feature_dim, float* out);

/* ------------------------------------------------------------------------
 * Toy-model path (the reference's own model, fp64, bit-exact to its CPU).
 * Ranks are CUDA streams on the current device; each rank runs exactly its
 * plan range, as WorkerGroup's OpenMP threads do upstream.
 * ------------------------------------------------------------------------ */

/* Replaces WorkerGroup::parallel_encode (engine.hpp:85-86, engine.cpp:78-101)
 * and, with sp_degree = 1 and one range [0,F), serial_encode (engine.cpp:52-57).
 *   enc_w      host, d*p row-major (EncoderParams::w, policy.hpp:17-23)
 *   frames     host, n_frames*p (Video::frames[i].features concatenated)
 *   ranges     host, 2*sp_degree (a ShardPlan covering n_frames)
 *   out        host, n_frames*d, frame-major: the all-gathered embeddings
 *   rank_items host, sp_degree: frames encoded by each rank (encoder_invocations)
 * Errors mirror engine.cpp:80-83 ("parallel_encode: plan does not cover the
 * video frames", "parallel_encode: plan degree mismatch") and policy.cpp:37-38. */
mrsp_status mrsp_toy_encode(int sp_degree, const double* enc_w, int d, int p,
                            const double* frames, uint64_t n_frames, const uint64_t* ranges,
                            double* out, uint64_t* rank_items);

/* Replaces WorkerGroup::parallel_prefill (engine.hpp:91-94, engine.cpp:103-130)
 * and serial_prefill (engine.cpp:59-71).
 *   theta      host, PolicyParams::theta with the policy.hpp:39-53 layout
 *              E_txt(V*d) | A(h*d) | B(h*d) | c(h) | U(V*h) | b(V)
 *   contexts   host, n_rows*d
 *   rows       host, n_rows*max_len padded token ids (PaddedBatch::rows)
 *   lengths    host, n_rows true lengths
 *   ranges     host, 2*sp_degree (a ShardPlan over max_len)
 *   out        host, (sum lengths)*V logits, row-major over real positions
 *   pad_reads  host, 1: number of reads past a row's true length (always 0)
 * prev = EOS (1) at t = 0, else rows[r][t-1] (engine.cpp:124). */
mrsp_status mrsp_toy_prefill(int sp_degree, const double* theta, int V, int d, int h,
                             const double* contexts, const int32_t* rows,
                             const uint64_t* lengths, uint64_t n_rows, uint64_t max_len,
                             const uint64_t* ranges, double* out, uint64_t* pad_reads);

/* Backward of the toy policy: grpo_gradient
 * (grpo.cpp:122-206 over GradAccumulator, policy.cpp:195-260) and
 * sft_loss_and_grad (grpo.cpp:208-223) on the device. Replaces those two
 * reference functions (grpo.hpp:52-62) for a sequence given as its frame
 * embeddings + text tokens (MultimodalSequence, mmseq.hpp).
 *   theta, ref    host, param_count(V, d, h) doubles each (policy.hpp:39-56)
 *   frame_emb     host, n_frames x d;  text_tokens host, n_text
 *   tokens        host, the rollouts' tokens concatenated (sum(lengths));
 *                 old_logprobs likewise; advantages host, n_rollouts
 *   ranges        host, 2 * sp_degree: ShardPlan over the longest rollout's
 *                 positions (as mrsp_toy_prefill); rank w runs the positions
 *                 t in [b_w, e_w) of every rollout
 *   grad          host out, param_count doubles
 *   stats         host out, 4: objective, mean_kl, clip_fraction, token_count
 * The position terms run sharded; the parameter sums run in the reference's
 * serial (rollout, t) order, so every sp_degree returns the same bits.
 * Errors: empty group / rollout / targets, token or text token out of range,
 * empty sequence -> MRSP_INVALID_ARGUMENT. */
mrsp_status mrsp_toy_grpo_gradient(int sp_degree, const double* theta, const double* ref, int V,
                                   int d, int h, const double* frame_emb, uint64_t n_frames,
                                   const int32_t* text_tokens, uint64_t n_text,
                                   const int32_t* tokens, const uint64_t* lengths,
                                   uint64_t n_rollouts, const double* old_logprobs,
                                   const double* advantages, double clip_eps, double kl_beta,
                                   int sampled_kl, const uint64_t* ranges, double* grad,
                                   double* stats);
/* loss: host out, 1 (mean teacher-forced cross-entropy); ranges over n_targets */
mrsp_status mrsp_toy_sft_loss_and_grad(int sp_degree, const double* theta, int V, int d, int h,
                                       const double* frame_emb, uint64_t n_frames,
                                       const int32_t* text_tokens, uint64_t n_text,
                                       const int32_t* targets, uint64_t n_targets,
                                       const uint64_t* ranges, double* loss, double* grad);

/* ------------------------------------------------------------------------
 * Device operators of the transformer-shaped path (dev pointers, async on
 * `stream`). They are the building blocks the engine below chains; exported
 * so the parity tests can check each kernel in isolation.
 * ------------------------------------------------------------------------ */
typedef enum {
  GEMM_EPI_STORE_BF16 = 0,     /* C = A.B^T                                 */
  GEMM_EPI_BIAS_BF16 = 1,      /* C = A.B^T + bias                          */
  GEMM_EPI_BIAS_GELU_BF16 = 2, /* C = gelu_tanh(A.B^T + bias)               */
  GEMM_EPI_RESID_F32 = 3,      /* resid(fp32) += A.B^T (+ bias)             */
  GEMM_EPI_SWIGLU_BF16 = 4,    /* per 256-col tile [gate128|up128]:
                                  C[:, tile*128 + j] = silu(g_j) * u_j      */
  GEMM_EPI_STORE_F32 = 5,      /* C(fp32) = A.B^T (+ bias)                  */
  GEMM_EPI_LOGPROB_PARTIAL = 6, /* internal: LM-head tile (max, sumexp, target) */
  GEMM_EPI_QKV_SCATTER = 7,     /* internal: +bias, bf16, RoPE on q/k heads, each 128-col
                                   head block stored to its owner rank(s) (fused Ulysses
                                   sequence -> head all-to-all)                           */
  GEMM_EPI_SWIGLU_BWD = 8       /* internal (backward): per 256-col tile [gate128|up128]
                                   with dA = the gradient of the SwiGLU output: C = [dA u
                                   silu'(g) | dA silu(g)] (bf16, same interleave as the
                                   weight rows) and the forward output silu(g) u again   */
} mrsp_gemm_epilogue;

/* tcgen05 BF16 GEMM, fp32 accumulate: A[M][lda], B[N][ldb] (both K-major),
 * C per epilogue. K, lda, ldb multiples of 8. Replaces the per-position
 * scalar contractions of hidden_state/step_logits (policy.cpp:85-119) and
 * encode_frame (policy.cpp:36-47) in the transformer-shaped model. */
mrsp_status mrsp_op_gemm_bf16(const void* A, const void* B, void* C, int M, int N, int K, int lda,
                              int ldb, int ldc, int epilogue, const float* bias, float* resid,
                              int ldr, void* stream);

/* Same GEMM with MN-major operands, for the backward pass (grpo.cpp:122-223
 * turned into a transformer backward): a_mn = 1 means A is stored [K][lda]
 * (element (m, k) at A[k*lda + m]); b_mn = 1 means B is stored [K][ldb].
 * dgrad dX = dY . W reads the weight W[N_out][K_in] with b_mn = 1; wgrad
 * dW = dY^T . X reads both token-major activations with a_mn = b_mn = 1 (K =
 * tokens, any count). Epilogues STORE_BF16 / BIAS_BF16 / STORE_F32 /
 * RESID_F32. */
mrsp_status mrsp_op_gemm_bf16_mn(const void* A, const void* B, void* C, int M, int N, int K,
                                 int lda, int ldb, int ldc, int a_mn, int b_mn, int epilogue,
                                 const float* bias, float* resid, int ldr, void* stream);

/* Same GEMM with a split-K workspace (device, fp32): when M <= 128 and the
 * N tiles cannot fill the SMs (the decode steps' G-row projections), K is
 * split across CTAs, fp32 partials land in the workspace and a second kernel
 * sums them in split order and applies the epilogue (deterministic).
 * mrsp_gemm_splitk_workspace_bytes(M) bytes let every such GEMM split fully;
 * a smaller workspace (or none) just splits less. Plain epilogues only
 * (STORE/BIAS/GELU/RESID/SWIGLU/STORE_F32). */
mrsp_status mrsp_op_gemm_bf16_splitk(const void* A, const void* B, void* C, int M, int N, int K,
                                     int lda, int ldb, int ldc, int epilogue, const float* bias,
                                     float* resid, int ldr, void* workspace, size_t ws_bytes,
                                     void* stream);
size_t mrsp_gemm_splitk_workspace_bytes(int M);

/* Fused vocabulary projection + log-softmax + gather (north-star item 5):
 *   logprob[i] = log_softmax(X[i] . W^T)[targets[i]],  lse[i] = logsumexp(X[i] . W^T)
 * X [M][ldx] bf16 (final-normed hidden at scored positions), W [V][K] bf16.
 * The [M x V] logits are never written to memory: each 128x256 tile's
 * (max, sum exp) and the target logit are reduced in the GEMM epilogue, then
 * combined across vocab tiles. lse may be NULL. Replaces log_softmax
 * (common.hpp:95-104) + the gather lp[y] (grpo.cpp:82-85, policy.cpp:159-174)
 * over materialised logits (engine.hpp:88-94). Workspace from
 * mrsp_lmhead_workspace_bytes(M, V). */
size_t mrsp_lmhead_workspace_bytes(int M, int V);
mrsp_status mrsp_op_lmhead_logprob(const void* X, int ldx, const void* W, int M, int V, int K,
                                   const int32_t* targets, float* logprob, float* lse,
                                   void* workspace, size_t ws_bytes, void* stream);

/* Fused policy + reference LM head: for each scored token
 * one vocabulary sweep over both models yields log pi_theta(y), log pi_ref(y)
 * and the exact KL(pi_theta || pi_ref) = sum_v p_v (log p_v - log q_v) — the
 * quantities evaluate_from_logits computes from two materialised logit
 * tensors (grpo.cpp:68-108, exact KL at :94-96; policy.cpp:176-193).
 * X_* [M][K] bf16 (final-normed hidden of each model), W_* [V][K] bf16. */
size_t mrsp_lmhead_dual_workspace_bytes(int M, int V);
mrsp_status mrsp_op_lmhead_dual(const void* X_policy, const void* W_policy, const void* X_ref,
                                const void* W_ref, int M, int V, int K, const int32_t* targets,
                                float* logprob_policy, float* logprob_ref, float* kl,
                                void* workspace, size_t ws_bytes, void* stream);

/* GRPO token terms (evaluate_from_logits, grpo.cpp:68-108) over per-token
 * device vectors in (rollout, position) order: log pi_theta(y), log pi_old(y),
 * log pi_ref(y) (sampled_kl) or the exact per-token KL (from
 * mrsp_op_lmhead_dual), per-rollout advantages and lengths. out4 (device,
 * fp64) = [objective, mean_kl, clip_fraction, token_count]. */
mrsp_status mrsp_op_grpo_stats(const float* logprob, const float* old_logprob,
                               const float* ref_logprob, const float* kl, const float* advantages,
                               const int32_t* lengths, int G, double clip_eps, double kl_beta,
                               int sampled_kl, double* out4, void* stream);

/* RMSNorm (Qwen2): out[i] = bf16(w * x[rows ? rows[i] : i] * rsqrt(mean(x^2) + eps)),
 * x fp32 [.][ldx], out bf16 [n][ldo]. */
mrsp_status mrsp_op_rmsnorm(const float* x, int ldx, const float* w, void* out, int ldo, int n,
                            int d, float eps, const int32_t* rows, void* stream);
/* LayerNorm (SigLIP): out = bf16((x - mean) * rsqrt(var + eps) * w + b). */
mrsp_status mrsp_op_layernorm(const float* x, int ldx, const float* w, const float* b, void* out,
                              int ldo, int n, int d, float eps, void* stream);
/* Rotate-half RoPE in place on n_heads 128-dim heads starting at column col0
 * of bf16 rows, angle = fp32(pos) * fp32(theta^(-2i/128)). */
mrsp_status mrsp_op_rope(void* qkv, int ld, int col0, int n_heads, const int32_t* pos, int n,
                         float theta, void* stream);
/* Pixels [F][3][H][W] fp32 -> patch rows bf16 [F*(H/P)*(W/P)][kpad], zero padded. */
mrsp_status mrsp_op_patchify(const float* pixels, void* out, int F, int H, int W, int P, int kpad,
                             void* stream);
/* MR-SP packed-sequence builder for global positions [p0, p0 + n): hidden fp32
 * rows gathered from frame embeddings / the token embedding table, position
 * ids and the pad mask. Layout: [n_frame_tok frame tokens | n_q question |
 * G rows x Lmax], row g = [EOS, resp[g][0 .. len_g - 2], PAD ...]
 * (pad_batch, engine.cpp:31-43; prev = EOS at t = 0, engine.cpp:124). */
mrsp_status mrsp_op_pack_sequence(const void* frame_emb, int n_frame_tok, const int32_t* question,
                                  int n_q, const int32_t* resp, const int32_t* lengths, int Lmax,
                                  const void* embed, int d, int64_t p0, int n, float* hidden,
                                  int32_t* pos_ids, uint8_t* pad_mask, int32_t* tokens,
                                  void* stream);

typedef enum {
  ATTN_CAUSAL_PREFIX = 0, /* k <= q && (k < Lp || row(k) == row(q)), row(x) = (x-Lp)/Lmax */
  ATTN_BLOCK_DIAG = 1     /* q / blk == k / blk (bidirectional within a frame)          */
} mrsp_attn_mask;

/* tcgen05 flash-attention forward, head dim 128, bf16 in/out, fp32 softmax.
 * Query head h reads Q columns [q_col0 + 128h, +128) and kv head h / q_per_kv
 * of K/V; writes O columns [o_col0 + 128h, +128). L rows (tokens). The
 * CAUSAL_PREFIX mask is the MR-SP packed GRPO group: the shared prompt prefix
 * (video + question, Lp tokens) followed by G rollout rows padded to Lmax.
 * Replaces the prefix pooling of context_vector (policy.cpp:63-80) that the
 * reference shares across the G rows (grpo.cpp:53). */
mrsp_status mrsp_op_attention(const void* Q, int ldq, int q_col0, const void* K, int ldk,
                              int k_col0, const void* V, int ldv, int v_col0, void* O, int ldo,
                              int o_col0, int L, int n_heads, int q_per_kv, float scale, int mode,
                              int Lp, int Lmax, int blk, void* stream);

/* Backward-pass operators (grpo.cpp:122-223 carried through
 * the transformer-shaped model). Same argument conventions as above.
 *
 * Attention forward that also writes the per-(head, row) log-sum-exp the
 * backward needs: lse[h*lse_ld + q] = log2 sum_k 2^(s_qk * scale * log2 e). */
mrsp_status mrsp_op_attention_lse(const void* Q, int ldq, int q_col0, const void* K, int ldk,
                                  int k_col0, const void* V, int ldv, int v_col0, void* O,
                                  int ldo, int o_col0, int L, int n_heads, int q_per_kv,
                                  float scale, int Lp, int Lmax, float* lse, int lse_ld,
                                  void* stream);
/* Attention backward (MR-SP causal-prefix mask, head dim 128): qkv [L][ld_qkv]
 * post-RoPE (q heads at q_col0 + 128h, kv heads at k_col0 / v_col0 + 128g),
 * O / dO [L][..] (head h at 128h), lse from mrsp_op_attention_lse, D a
 * [n_heads][ld_stat] fp32 workspace; dq / dk / dv land in dqkv at the qkv
 * column layout. Deterministic (no atomics). */
mrsp_status mrsp_op_attention_bwd(const void* qkv, int ld_qkv, int q_col0, int k_col0, int v_col0,
                                  const void* O, int ld_o, const void* dO, int ld_do,
                                  const float* lse, float* D, int ld_stat, void* dqkv,
                                  int ld_dqkv, int L, int n_heads, int q_per_kv, float scale,
                                  int Lp, int Lmax, void* stream);
/* RMSNorm backward: dx_acc[row] += dL/dx (x fp32, dy fp32), dw_out[d] += dL/dw
 * (may be NULL); rows (may be NULL) maps row i of dy to the x / dx_acc row. */
mrsp_status mrsp_op_rmsnorm_bwd(const float* x, int ldx, const float* w, const float* dy, int ldy,
                                float* dx_acc, int ld_dx, int n, int d, float eps,
                                const int32_t* rows, float* dw_out, void* stream);
/* SwiGLU backward fused into the gate/up GEMM (GEMM_EPI_SWIGLU_BWD): X [M][K],
 * W_gu [N][K] ([gate128 | up128] row blocks), dA [M][N/2] -> dGU [M][N] and the
 * forward output act [M][N/2] (bf16). */
mrsp_status mrsp_op_gemm_swiglu_bwd(const void* X, const void* W_gu, const void* dA, void* dGU,
                                    void* act, int M, int N, int K, void* stream);
/* dJ/dlogits of the GRPO objective from both models' final hidden rows, one
 * vocabulary tile at a time (never the [M x V] fp32 logits):
 * G[t][v] = pi (kw (lp - lq - kl_t) - coef_t) + coef_t [v == y_t], bf16 [M][ldg].
 * lse_*: per-row log-partitions (natural log). */
mrsp_status mrsp_op_lmhead_dual_dlogits(const void* X_policy, const void* W_policy,
                                        const void* X_ref, const void* W_ref, int M, int V, int K,
                                        const int32_t* targets, const float* coef, float kw,
                                        const float* kl, const float* lse_policy,
                                        const float* lse_ref, void* G, int ldg, void* stream);

/* ------------------------------------------------------------------------
 * The MR-SP engine (transformer-shaped model; BASELINE.json configs c1..c5).
 *
 * Stage 1 — replaces WorkerGroup::parallel_encode + all_gather +
 *   EmbeddingCache::get_or_encode (engine.cpp:78-101, :132-197): frames are
 *   sharded with plan_shards(F, sp), each rank runs the SigLIP-shaped tower +
 *   projector on its frames (tcgen05 GEMMs, block-diagonal attention), the
 *   embeddings are all-gathered (NCCL over NVLink, or in-process) into a
 *   device-resident cache keyed by video id with the reference's exactly-once
 *   fill protocol and counters.
 * Stage 2 — replaces pad_batch + plan_shards(max_len) + parallel_prefill +
 *   log_softmax/gather (engine.cpp:31-43, :103-130; grpo.cpp:44-55, :82-85):
 *   the GRPO group is packed as [video | question | G rows padded to Lmax],
 *   sharded with plan_shards(L_total, sp), and prefilled through a
 *   Qwen2.5-shaped decoder with Ulysses all-to-all around the attention; the
 *   fused LM head returns per-token log-probs of the response tokens.
 *
 * Ranks: sp_degree = n_procs x local ranks. n_procs == 1 runs sp_degree
 * virtual ranks on the current device (loopback collectives); n_procs > 1
 * requires sp_degree == n_procs, one process per GPU, and a NCCL unique id
 * broadcast by the launcher (mrsp_nccl_unique_id on rank 0).
 * ------------------------------------------------------------------------ */
typedef struct {
  int image_size;  /* 224 (c2..c5) / 64 (c1)                     */
  int patch;       /* 14 / 8  -> tokens per frame (image/patch)^2   */
  int v_dim;       /* 1152 / 256                                    */
  int v_heads;     /* 16 / 4                                        */
  int v_head_dim;  /* 72 / 64 (<= 128; padded to 128 on device)     */
  int v_mlp;       /* 4304 / 1024                                   */
  int v_layers;    /* 27 / 2                                        */
  int dim;         /* 3584 / 256                                    */
  int n_q_heads;   /* 28 / 4                                        */
  int n_kv_heads;  /* 4 / 2                                         */
  int head_dim;    /* 128 (the only supported value)                */
  int mlp;         /* 18944 / 1024 (multiple of 128)                */
  int layers;      /* 28 (c3..c5) / 4 (c2) / 2 (c1)                 */
  int vocab;       /* 152064 / 32                                   */
  float rope_theta;
  float rms_eps;
  float ln_eps;
} mrsp_model_config;

typedef struct mrsp_engine mrsp_engine;

/* Ulysses plan of SP rank `rank` (host function; the engine's all-to-all uses
 * exactly this): out14 = [q_lo, q_hi, kv_lo, kv_hi, q_per_kv, then for Q, K, V
 * the (src col, dst col, width) block a sequence shard sends this rank]. For
 * sp <= n_kv heads split contiguously; for sp > n_kv each kv head is replicated
 * to sp/n_kv ranks that split its query-head group with plan_shards. */
mrsp_status mrsp_ulysses_plan(int n_q, int n_kv, int sp, int rank, int32_t* out14);
/* The engine's head split of SP rank `rank` (row_split != 0: the peer-memory
 * transports' query-row split when sp > n_kv): out7 = {q_lo, q_hi, kv_lo,
 * kv_hi, q_per_kv, row_parts, row_part}. */
mrsp_status mrsp_head_split(int n_q, int n_kv, int sp, int rank, int row_split, int32_t* out7);

/* Query-row split used instead by the peer-memory / virtual-rank transports
 * when sp > n_kv (MRSP_ULYSSES_SPLIT=heads restores the head split above):
 * the m = sp / n_kv ranks sharing kv head g = rank / m each hold all n_q/n_kv
 * of its query heads and compute the 256-row query blocks b of n_blocks =
 * ceil(L / 256) with mrsp_attn_row_part(b, n_blocks, m) == rank % m — blocks
 * dealt heaviest-first (causal cost grows with b) in a snake, so the m shares
 * of attention work differ by at most one block. Returns -1 on bad input. */
int mrsp_attn_row_part(int block, int n_blocks, int m);

/* Rollout generation (policy.cpp:121-157 sample_rollout):
 * G rows sampled from the policy after the prompt [cached video | question]:
 * one prompt prefill keeps every layer's K/V, then each decode step runs the G
 * rows through the LLM (decode attention over the prompt K/V and the row's own
 * keys) and samples token t of every unfinished row with probability
 * softmax(logits / temperature), u = splitmix64-hash(seed, row, t) in [0, 1);
 * a row stops after EOS (1). Outputs: tokens [G][max_len] (PAD = 0 after the
 * end), lengths [G] (EOS included), old_logprobs [G][max_len] =
 * log_softmax(logits)[token] at temperature 1. SP > 1 (virtual ranks or one
 * process per GPU over peer memory; not the NCCL transport): the prompt
 * prefill is sequence-parallel, every rank gathers the prompt K/V of all kv
 * heads from the ranks' head shards and runs the decode — the outputs are
 * bit-identical on every rank and to SP = 1 (grpo.cpp:376-386 generates the G
 * rollouts inside the SP engine loop). */
mrsp_status mrsp_engine_generate(mrsp_engine* e, const char* video_id, const int32_t* question,
                                 int n_q, int G, int max_len, float temperature, uint64_t seed,
                                 int32_t* tokens_out, int32_t* lengths_out,
                                 float* old_logprobs_out);

/* GRPO gradient of the policy LLM through the MR-SP prefill (
 * grpo_gradient, grpo.cpp:122-206, with the exact or k3 KL): the video must
 * be encoded (mrsp_engine_encode / _step). Runs the reference and policy
 * passes, the fused dual LM head, then the backward of the LM head and every
 * decoder layer (recomputed from its kept input) into fp32 gradients held by
 * the engine (mrsp_engine_save_grads). Memory per rank: the fp32 layer inputs
 * (layers x shard tokens x dim x 4 bytes) and, when the largest rank's share
 * fits in a quarter of the device, each layer's attention output and
 * log-sum-exp so the recompute skips the attention (env MRSP_BWD_STASH_ATTN =
 * 0 / 1: never / always; the gradients are bit-identical either way). old_logprobs: sum(lengths) host floats
 * (row-major), advantages: G host floats; stats4 (host) = {objective, mean_kl,
 * clip_fraction, token_count}; logprob_policy (host, may be NULL). Any SP
 * degree (virtual ranks, or one process per GPU on the peer-memory transport,
 * where every rank of the group makes the same call: it is collective); the
 * vision tower and projector are frozen. */
mrsp_status mrsp_engine_grpo_backward(mrsp_engine* e, const char* video_id,
                                      const int32_t* question, int n_q, const int32_t* resp,
                                      const int32_t* lengths, int G, int Lmax,
                                      const float* old_logprobs, const float* advantages,
                                      double clip_eps, double kl_beta, int sampled_kl,
                                      double* stats4, float* logprob_policy);
/* SFT loss and gradient (sft_loss_and_grad, grpo.cpp:208-223) of the policy
 * LLM over the G teacher-forced rows of a group (the reference's single target
 * row is G = 1): loss = mean over all row tokens of -log pi(y), written to
 * loss_out (host); gradients of the loss kept like mrsp_engine_grpo_backward's;
 * logprob_policy (host, may be NULL). */
mrsp_status mrsp_engine_sft_backward(mrsp_engine* e, const char* video_id, const int32_t* question,
                                     int n_q, const int32_t* resp, const int32_t* lengths, int G,
                                     int Lmax, double* loss_out, float* logprob_policy);
/* The last mrsp_engine_grpo_backward's gradients as F32 safetensors under the
 * policy's tensor names (model.layers.N.*, model.embed_tokens.weight, ...). */
mrsp_status mrsp_engine_save_grads(mrsp_engine* e, const char* path);

/* Weights as safetensors with Hugging Face tensor names (SigLIP
 * vision_model.*, projector mm_projector.{0,2}.*, Qwen2 model.* / lm_head.weight;
 * the GRPO reference model is saved with the prefix "ref."), unpadded HF shapes.
 * load: part 0 = vision tower + projector, 1 = policy LLM, 2 = reference LLM,
 * reading the names under `prefix` ("" or e.g. "ref."); BF16 and F32 tensors are
 * converted to the engine's storage type; a missing tensor or a shape that does
 * not match the engine geometry is MRSP_INVALID_ARGUMENT. */
mrsp_status mrsp_engine_save_weights(mrsp_engine* e, const char* path);
mrsp_status mrsp_engine_load_weights(mrsp_engine* e, const char* path, int part,
                                     const char* prefix);

/* Embedding-cache persistence: write a cached (encoded) video's gathered
 * embeddings to `path`; load them under `video_id` so later fetches hit without
 * encoding (the file records frames, tokens/frame, dim and an encoder-geometry
 * fingerprint; a mismatch is MRSP_INVALID_ARGUMENT). */
mrsp_status mrsp_engine_cache_save(mrsp_engine* e, const char* video_id, const char* path);
mrsp_status mrsp_engine_cache_load(mrsp_engine* e, const char* video_id, const char* path,
                                   int* frames_out);

/* Peer-memory transport (one process per GPU, no NCCL): create the engine with
 * n_procs > 1 and nccl_id = NULL, then on every rank
 *   mrsp_engine_p2p_export(e, max_frames, max_tokens, max_scored, blob)   -> blob
 *   (all-gather the n_procs blobs in rank order on the host)
 *   mrsp_engine_p2p_import(e, blobs)
 * Each rank exports fixed landing buffers (its head shard of the packed
 * sequence, its sequence shard of attention output, the gathered video, the
 * group outputs) through CUDA IPC; the fused QKV / attention epilogues and the
 * gathers store straight into peers' buffers over NVLink, ordered by a device
 * barrier. Capacities bound the video (frames), the packed sequence (tokens)
 * and the scored tokens of every later call. */
size_t mrsp_p2p_blob_bytes(void);
mrsp_status mrsp_engine_p2p_export(mrsp_engine* e, int max_frames, long max_tokens,
                                   long max_scored, void* blob_out);
mrsp_status mrsp_engine_p2p_import(mrsp_engine* e, const void* blobs);

/* Fills the 128-byte NCCL unique id (call on rank 0, broadcast to all). */
mrsp_status mrsp_nccl_unique_id(void* out128);

/* Creates the engine on the current device and initialises synthetic weights
 * (counter-based uniform init, see oracle/transformer.py). with_ref = 0 makes
 * the reference model alias the policy (the reference bench's behaviour,
 * engine.cpp:218-219). */
mrsp_status mrsp_engine_create(const mrsp_model_config* cfg, int sp_degree, int proc_rank,
                               int n_procs, uint64_t vision_seed, uint64_t policy_seed,
                               uint64_t ref_seed, int with_ref, const void* nccl_id,
                               mrsp_engine** out);
mrsp_status mrsp_engine_destroy(mrsp_engine* e);

/* Stage 1: encode + gather the video into the cache (or hit it).
 * pixels: F x 3 x S x S fp32, host or device (pixels_on_device). hit: 0/1.
 * use_cache = 0 encodes without touching the cache (cache-off bench cell). */
mrsp_status mrsp_engine_encode(mrsp_engine* e, const char* video_id, const float* pixels, int F,
                               int pixels_on_device, int use_cache, int* hit);

/* Stage 2: per-token log-probs of G rollouts against the cached video
 * `video_id`. resp: G x Lmax token ids (row g valid below lengths[g]);
 * model 0 = policy, 1 = reference. logprob/lse: sum(lengths) floats in
 * row-major (rollout, position) order; host memory unless out_on_device. */
mrsp_status mrsp_engine_prefill_logprobs(mrsp_engine* e, const char* video_id,
                                         const int32_t* question, int n_q, const int32_t* resp,
                                         const int32_t* lengths, int G, int Lmax, int model,
                                         float* logprob, float* lse, int out_on_device);

/* One MR-SP step (engine.cpp:203-225 contract): G embedding fetches (cache
 * on: 1 miss + G-1 hits), then policy and reference prefill; the two LM heads
 * run as one fused sweep that also yields the exact per-token KL (kl may be
 * NULL). Outputs: sum(lengths) floats each, host unless out_on_device. */
mrsp_status mrsp_engine_step(mrsp_engine* e, const char* video_id, const float* pixels, int F,
                             int pixels_on_device, int use_cache, const int32_t* question,
                             int n_q, const int32_t* resp, const int32_t* lengths, int G,
                             int Lmax, float* logprob_policy, float* logprob_ref, float* kl,
                             int out_on_device);

/* Counters: [encoder_invocations, cache_hits, cache_misses, gather_bytes,
 * pad_reads, a2a_bytes] (EngineStats, engine.hpp:27-41, plus a2a bytes). */
mrsp_status mrsp_engine_stats(mrsp_engine* e, uint64_t* out6, int reset);
mrsp_status mrsp_engine_cache(mrsp_engine* e, int op /*0 size,1 clear,2 set capacity*/, int arg,
                              uint64_t* size_out);
/* Copies the cached [F*T][dim] bf16 embeddings of video_id to host_out, which
 * holds capacity_bytes (MRSP_INVALID_ARGUMENT when too small; nothing is
 * written). frames_out (may be NULL) receives F; host_out == NULL only queries F. */
mrsp_status mrsp_engine_get_embeddings(mrsp_engine* e, const char* video_id, void* host_out,
                                       size_t capacity_bytes, int* frames_out);
/* Per-kernel-class CUDA-event timing: cls 0 LLM attention, 1 LLM GEMMs,
 * 2 vision tower, 3 LM head, 4 collectives, 5 norms/rope/pack. */
mrsp_status mrsp_engine_profile(mrsp_engine* e, int enable, int cls, double* ms, int64_t* launches);
/* The stream the engine launches on (cudaStream_t). */
void* mrsp_engine_stream(mrsp_engine* e);

#ifdef __cplusplus
}
#endif
#endif /* MRSP_C_H_ */
