// misc.h — HBM-bound kernels around the tensor-core work (csrc/kernels_misc.cu).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace mrsp {

void rmsnorm(const float* x, int ldx, const float* w, __nv_bfloat16* out, int ldo, int n, int d,
             float eps, const int* rows, cudaStream_t s);
void layernorm(const float* x, int ldx, const float* w, const float* b, __nv_bfloat16* out,
               int ldo, int n, int d, float eps, cudaStream_t s);
void rope_inv_freq(float theta, float* inv64);  // HF float32 convention
void set_rope_inv_freq(const float* inv_freq64, cudaStream_t s);
void rope(__nv_bfloat16* qkv, int ld, int col0, int n_heads, const int* pos, int n, cudaStream_t s);
void patchify(const float* pix, __nv_bfloat16* out, int F, int H, int W, int P, int kpad,
              cudaStream_t s);
void broadcast_rows(const float* src, float* dst, int n, int period, int d, cudaStream_t s);
void pack_sequence(const __nv_bfloat16* frame_emb, int n_frame_tok, const int* question, int n_q,
                   const int* resp, const int* lengths, int Lmax, const __nv_bfloat16* embed,
                   int d, long p0, int n, float* hidden, int* pos_ids, unsigned char* pad_mask,
                   int* tok_out, cudaStream_t s);
void logprob_combine(const float2* part, int n_tiles, const float* tgt_logit, int n, float* lp,
                     float* lse, cudaStream_t s);
void init_uniform_bf16(__nv_bfloat16* w, size_t n, uint64_t key, float scale, cudaStream_t s);
void init_uniform_f32(float* w, size_t n, uint64_t key, float scale, float offset, cudaStream_t s);
void convert_bf16_f32(const __nv_bfloat16* in, float* out, size_t n, cudaStream_t s);

// rollout generation (csrc/decode.cu)
size_t decode_partial_bytes(int max_prefix, int max_len, int G, int n_kv);
// The prompt K/V is head-major, [n_kv][K | V][Lp][128]; the row cache of
// generated tokens is [rows][ld_kv] (K heads | V heads at v_off).
// maps: optional TMA descriptors {prompt K/V, row cache} built once per
// generation (decode_tensor_maps) so a step encodes none
bool decode_use_tensor_cores(int Lp);
void decode_tensor_maps(const void* kv_prefix, int Lp, int n_kv, const void* kv_rows, long rows,
                        int ld_kv, void* maps_out /* 2 x CUtensorMap */);
// Decode steps read the step index t from device memory (`tdev`), so one
// captured CUDA graph of a step replays for every t; host-side `t_grid` only
// sizes the attention grid (the current t eagerly, max_len - 1 in a graph:
// chunks past the live row keys write empty partials). max_rows (max_len x G)
// sizes the chunks, so eager and graph steps split the keys identically.
void decode_attention(const void* q, int ldq, int q_col0, const void* kv_prefix,
                      const void* kv_rows, int ld_kv, int v_off, int Lp, int G, int t_grid,
                      int max_rows, const int* tdev, int q_per_kv, int n_kv, float scale,
                      float* part, void* out, int ldo, cudaStream_t s, const void* maps = nullptr);
// norm_w non-null: also out = RMSNorm(hidden) (the first layer's attention norm)
void decode_embed(const __nv_bfloat16* embed, int d, const int* tokens, int max_len,
                  const int* tdev, int G, int pos_base, float* hidden, int* pos_out, cudaStream_t s,
                  const float* norm_w = nullptr, __nv_bfloat16* norm_out = nullptr,
                  float eps = 0.f);
// rows[t * G + g][0, kvw) = qkv[g][col0, col0 + kvw) (this step's K | V per row)
void decode_append_kv(const __nv_bfloat16* qkv, int ldq, int col0, __nv_bfloat16* rows, int kvw,
                      int G, const int* tdev, cudaStream_t s);
size_t sample_workspace_bytes(int G);
void sample_tokens(const float* logits, int G, int V, float temperature, uint64_t seed,
                   const int* tdev, int* done, int* tokens, float* old_lp, int* lengths,
                   int max_len, void* ws /* sample_workspace_bytes(G) */, cudaStream_t s);
void decode_step_advance(int* tdev, cudaStream_t s);

}  // namespace mrsp
