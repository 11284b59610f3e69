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
/* Number of visible CUDA devices (0 when none); never fails. */
int mrsp_device_count(void);

/* ------------------------------------------------------------------------
 * Shard planning — replaces mrsp::plan_shards (engine.hpp:25, engine.cpp:15-29).
 * ranges receives 2*sp_degree values [b0,e0,b1,e1,...]. The first
 * (n mod k) ranges hold one extra item; empty ranges are legal.
 * MRSP_INVALID_ARGUMENT "plan_shards: sp_degree must be >= 1" when k < 1.
 * ------------------------------------------------------------------------ */
mrsp_status mrsp_plan_shards(uint64_t n_items, int sp_degree, uint64_t* ranges);

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
  GEMM_EPI_STORE_F32 = 5       /* C(fp32) = A.B^T (+ bias)                  */
} mrsp_gemm_epilogue;

/* tcgen05 BF16 GEMM, fp32 accumulate: A[M][lda], B[N][ldb] (both K-major),
 * C per epilogue. K, lda, ldb multiples of 8. Replaces the per-position
 * scalar contractions of hidden_state/step_logits (policy.cpp:85-119) and
 * encode_frame (policy.cpp:36-47) in the transformer-shaped model. */
mrsp_status mrsp_op_gemm_bf16(const void* A, const void* B, void* C, int M, int N, int K, int lda,
                              int ldb, int ldc, int epilogue, const float* bias, float* resid,
                              int ldr, void* stream);

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

#ifdef __cplusplus
}
#endif
#endif /* MRSP_C_H_ */
