// kernels_misc.cu — the HBM-bound kernels around the tensor-core work:
// norms, RoPE, patchify, the MR-SP sequence pack, the log-prob combine and the
// counter-based weight initialiser. All use 128-bit vector accesses on the
// contiguous (feature) dimension and grids sized as multiples of the SM count.
#include <cmath>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "common.h"
#include "misc.h"
#include "pdl.cuh"

namespace mrsp {
namespace {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---- RMSNorm (Qwen2): out = bf16(w * (x * rsqrt(mean(x^2) + eps))) ------------
// One warp per output row; optional row index map (gather) for the final norm
// over scored positions only.
__global__ void rmsnorm_kernel(const float* __restrict__ x, int ldx, const float* __restrict__ w,
                               __nv_bfloat16* __restrict__ out, int ldo, int n, int d, float eps,
                               const int* __restrict__ rows) {
  pdl_wait();
  pdl_trigger();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n) return;
  const int src = rows ? rows[warp] : warp;
  const float4* xr = reinterpret_cast<const float4*>(x + static_cast<size_t>(src) * ldx);
  float ss = 0.f;
  for (int i = lane; i < d / 4; i += 32) {
    const float4 v = xr[i];
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  ss = warp_sum(ss);
  const float r = rsqrtf(ss / static_cast<float>(d) + eps);
  const float4* wr = reinterpret_cast<const float4*>(w);
  __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>(out + static_cast<size_t>(warp) * ldo);
  for (int i = lane; i < d / 4; i += 32) {
    const float4 v = xr[i], g = wr[i];
    o[2 * i] = __floats2bfloat162_rn(g.x * (v.x * r), g.y * (v.y * r));
    o[2 * i + 1] = __floats2bfloat162_rn(g.z * (v.z * r), g.w * (v.w * r));
  }
}

// ---- LayerNorm (SigLIP): out = bf16((x - mu) * rsqrt(var + eps) * w + b) -------
__global__ void layernorm_kernel(const float* __restrict__ x, int ldx, const float* __restrict__ w,
                                 const float* __restrict__ b, __nv_bfloat16* __restrict__ out,
                                 int ldo, int n, int d, float eps) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n) return;
  const float4* xr = reinterpret_cast<const float4*>(x + static_cast<size_t>(warp) * ldx);
  float s = 0.f;
  for (int i = lane; i < d / 4; i += 32) {
    const float4 v = xr[i];
    s += v.x + v.y + v.z + v.w;
  }
  const float mu = warp_sum(s) / static_cast<float>(d);
  float q = 0.f;
  for (int i = lane; i < d / 4; i += 32) {
    const float4 v = xr[i];
    q += (v.x - mu) * (v.x - mu) + (v.y - mu) * (v.y - mu) + (v.z - mu) * (v.z - mu) +
         (v.w - mu) * (v.w - mu);
  }
  const float r = rsqrtf(warp_sum(q) / static_cast<float>(d) + eps);
  const float4* wr = reinterpret_cast<const float4*>(w);
  const float4* br = reinterpret_cast<const float4*>(b);
  __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>(out + static_cast<size_t>(warp) * ldo);
  for (int i = lane; i < d / 4; i += 32) {
    const float4 v = xr[i], g = wr[i], c = br[i];
    o[2 * i] = __floats2bfloat162_rn((v.x - mu) * r * g.x + c.x, (v.y - mu) * r * g.y + c.y);
    o[2 * i + 1] = __floats2bfloat162_rn((v.z - mu) * r * g.z + c.z, (v.w - mu) * r * g.w + c.w);
  }
}

// ---- RoPE (rotate-half, Qwen2) in place on the bf16 QKV rows ------------------
// heads [0, n_heads) of 128 dims starting at column col0; angle = fp32(pos) *
// inv_freq[i] (fp32 product, as the HF reference computes it), accurate sincos.
__constant__ float c_inv_freq[64];

__global__ void rope_kernel(__nv_bfloat16* __restrict__ qkv, int ld, int col0, int n_heads,
                            const int* __restrict__ pos, int n) {
  // thread = (row, frequency pair): bf16x2 accesses, one sincos pair reused
  // over every head of the row
  pdl_wait();
  pdl_trigger();
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n * 32) return;
  const int row = idx >> 5, i = (idx & 31) * 2;
  const float p = static_cast<float>(pos[row]);
  float sn0, cs0, sn1, cs1;
  sincosf(__fmul_rn(p, c_inv_freq[i]), &sn0, &cs0);
  sincosf(__fmul_rn(p, c_inv_freq[i + 1]), &sn1, &cs1);
  __nv_bfloat16* base = qkv + static_cast<size_t>(row) * ld + col0 + i;
  for (int h = 0; h < n_heads; ++h) {
    __nv_bfloat162* lo = reinterpret_cast<__nv_bfloat162*>(base + h * 128);
    __nv_bfloat162* hi = reinterpret_cast<__nv_bfloat162*>(base + h * 128 + 64);
    const float2 a = __bfloat1622float2(*lo), b = __bfloat1622float2(*hi);
    // explicit round-to-nearest ops (no FMA contraction): the fused QKV-scatter
    // GEMM epilogue computes the identical bits
    *lo = __floats2bfloat162_rn(__fsub_rn(__fmul_rn(a.x, cs0), __fmul_rn(b.x, sn0)),
                                __fsub_rn(__fmul_rn(a.y, cs1), __fmul_rn(b.y, sn1)));
    *hi = __floats2bfloat162_rn(__fadd_rn(__fmul_rn(b.x, cs0), __fmul_rn(a.x, sn0)),
                                __fadd_rn(__fmul_rn(b.y, cs1), __fmul_rn(a.y, sn1)));
  }
}

// ---- patchify: pixels [F][3][H][W] fp32 -> patches bf16 [F*T][kpad] ----------
// column c*P*P + ky*P + kx (the conv weight layout [dim][3][P][P]); zero pad.
// One CTA per (frame, patch row): the 3 x P x W input rows are staged in
// shared memory with coalesced float4 loads, then the W/P tokens' kpad-wide
// output rows (contiguous in HBM) are written with coalesced bf16x2 stores.
__global__ void patchify_kernel(const float* __restrict__ pix, __nv_bfloat16* __restrict__ out,
                                int F, int H, int W, int P, int kpad) {
  extern __shared__ float tile[];  // [3][P][W] staged rows, then [kpad] column -> tile offset
  const int gh = H / P, gw = W / P, PP = P * P, kreal = 3 * PP;
  const int f = blockIdx.x / gh, py = blockIdx.x % gh;
  int* koff = reinterpret_cast<int*>(tile + 3 * P * W);
  for (int k = threadIdx.x; k < kpad; k += blockDim.x)
    koff[k] = k < kreal ? ((k / PP) * P + (k / P) % P) * W + k % P : -1;
  for (int c = 0; c < 3; ++c) {
    const float* src = pix + ((static_cast<size_t>(f) * 3 + c) * H + py * P) * W;
    float* dst = tile + c * P * W;
    if ((W & 3) == 0) {
      for (int j = threadIdx.x; j < P * W / 4; j += blockDim.x)
        reinterpret_cast<float4*>(dst)[j] = reinterpret_cast<const float4*>(src)[j];
    } else {
      for (int j = threadIdx.x; j < P * W; j += blockDim.x) dst[j] = src[j];
    }
  }
  __syncthreads();
  __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>(
      out + (static_cast<size_t>(f) * gh * gw + static_cast<size_t>(py) * gw) * kpad);
  const int half = kpad / 2;
  for (int px = 0; px < gw; ++px) {
    const float* tp = tile + px * P;
    for (int k2 = threadIdx.x; k2 < half; k2 += blockDim.x) {
      const int o0 = koff[2 * k2], o1 = koff[2 * k2 + 1];
      o[px * half + k2] = __floats2bfloat162_rn(o0 >= 0 ? tp[o0] : 0.f, o1 >= 0 ? tp[o1] : 0.f);
    }
  }
}

// ---- rows[t] = src[t % period] (position embeddings broadcast over frames) ---
__global__ void broadcast_rows_kernel(const float* __restrict__ src, float* __restrict__ dst,
                                      int n, int period, int d) {
  const size_t total = static_cast<size_t>(n) * d / 4;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t row = i / (d / 4), c = i % (d / 4);
    reinterpret_cast<float4*>(dst)[i] =
        reinterpret_cast<const float4*>(src)[(row % period) * (d / 4) + c];
  }
}

// ---- MR-SP sequence pack ------------------------------------------------------
// Global packed layout: [frame tokens | question | G rows of
// Lmax], row i = [EOS, y_0 .. y_{len_i - 2}, PAD ...] (teacher forcing:
// engine.cpp:124 / policy.cpp:127 — prev = EOS at t = 0). For global
// positions [p0, p0 + n): hidden fp32 row, position id, pad flag.
__global__ void pack_kernel(const __nv_bfloat16* __restrict__ frame_emb, int n_frame_tok,
                            const int* __restrict__ question, int n_q,
                            const int* __restrict__ resp, const int* __restrict__ lengths, int Lmax,
                            const __nv_bfloat16* __restrict__ embed, int d, long p0, int n,
                            float* __restrict__ hidden, int* __restrict__ pos_ids,
                            unsigned char* __restrict__ pad_mask, int* __restrict__ tok_out) {
  const int Lp = n_frame_tok + n_q;
  for (int r = blockIdx.x; r < n; r += gridDim.x) {
    const long p = p0 + r;
    const __nv_bfloat16* src;
    int tok = -1, pos, pad = 0;
    if (p < n_frame_tok) {
      src = frame_emb + static_cast<size_t>(p) * d;
      pos = static_cast<int>(p);
    } else if (p < Lp) {
      tok = question[p - n_frame_tok];
      src = embed + static_cast<size_t>(tok) * d;
      pos = static_cast<int>(p);
    } else {
      const long q = p - Lp;
      const int row = static_cast<int>(q / Lmax), j = static_cast<int>(q % Lmax);
      const int len = lengths[row];
      if (j < len) {
        tok = j == 0 ? 1 /* Vocab::kEos */ : resp[static_cast<size_t>(row) * Lmax + j - 1];
      } else {
        tok = 0;  // Vocab::kPad
        pad = 1;
      }
      src = embed + static_cast<size_t>(tok) * d;
      pos = Lp + j;
    }
    if (threadIdx.x == 0) {
      pos_ids[r] = pos;
      pad_mask[r] = static_cast<unsigned char>(pad);
      if (tok_out) tok_out[r] = tok;
    }
    const __nv_bfloat162* s2 = reinterpret_cast<const __nv_bfloat162*>(src);
    float2* h2 = reinterpret_cast<float2*>(hidden + static_cast<size_t>(r) * d);
    for (int i = threadIdx.x; i < d / 2; i += blockDim.x) h2[i] = __bfloat1622float2(s2[i]);
  }
}

// ---- log-prob combine: lp = logit[target] - logsumexp over vocab tiles -------
__global__ void logprob_combine_kernel(const float2* __restrict__ part, int n_tiles,
                                       const float* __restrict__ tgt_logit, int n,
                                       float* __restrict__ lp, float* __restrict__ lse_out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n) return;
  const float2* pr = part + static_cast<size_t>(warp) * n_tiles;
  float m = -INFINITY;
  for (int t = lane; t < n_tiles; t += 32) m = fmaxf(m, pr[t].x);
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float s = 0.f;
  for (int t = lane; t < n_tiles; t += 32) s += pr[t].y * expf(pr[t].x - m);
  s = warp_sum(s);
  if (lane == 0) {
    const float lse = m + logf(s);
    lp[warp] = tgt_logit[warp] - lse;
    if (lse_out) lse_out[warp] = lse;
  }
}

// ---- counter-based synthetic weight init (bit-reproducible by the oracle) ----
// u = top 24 bits of splitmix64(key + i) / 2^24;  w = bf16(scale * (2u - 1))
__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__global__ void init_uniform_bf16_kernel(__nv_bfloat16* __restrict__ w, size_t n, uint64_t key,
                                         float scale) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const float u = static_cast<float>(splitmix64(key + i) >> 40) * 5.9604644775390625e-08f;
    w[i] = __float2bfloat16_rn(__fmul_rn(scale, __fadd_rn(__fmul_rn(2.0f, u), -1.0f)));
  }
}
__global__ void init_uniform_f32_kernel(float* __restrict__ w, size_t n, uint64_t key, float scale,
                                        float offset) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const float u = static_cast<float>(splitmix64(key + i) >> 40) * 5.9604644775390625e-08f;
    w[i] = __fadd_rn(offset, __fmul_rn(scale, __fadd_rn(__fmul_rn(2.0f, u), -1.0f)));
  }
}

__global__ void convert_bf16_f32_kernel(const __nv_bfloat16* __restrict__ in, float* __restrict__ out,
                                        size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    out[i] = __bfloat162float(in[i]);
}

int grid_for(size_t work, int threads) {
  static int sms = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  const size_t blocks = (work + threads - 1) / threads;
  return static_cast<int>(std::min<size_t>(std::max<size_t>(blocks, 1), static_cast<size_t>(sms) * 16));
}

}  // namespace

void rmsnorm(const float* x, int ldx, const float* w, __nv_bfloat16* out, int ldo, int n, int d,
             float eps, const int* rows, cudaStream_t s) {
  MRSP_REQUIRE(d % 4 == 0 && ldx % 4 == 0, MRSP_INVALID_ARGUMENT, "rmsnorm: d % 4");
  if (n <= 0) return;
  launch_pdl(rmsnorm_kernel, dim3((n + 7) / 8), dim3(256), 0, s, x, ldx, w, out, ldo, n, d, eps,
             rows);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

void layernorm(const float* x, int ldx, const float* w, const float* b, __nv_bfloat16* out,
               int ldo, int n, int d, float eps, cudaStream_t s) {
  MRSP_REQUIRE(d % 4 == 0 && ldx % 4 == 0, MRSP_INVALID_ARGUMENT, "layernorm: d % 4");
  if (n <= 0) return;
  layernorm_kernel<<<(n + 7) / 8, 256, 0, s>>>(x, ldx, w, b, out, ldo, n, d, eps);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

// RoPE inverse frequencies as HF transformers builds them (Qwen2
// RotaryEmbedding: 1.0 / base ** (arange(0, dim, 2).float() / dim)): float32
// exponent, float32 power (correctly rounded here), float32 reciprocal.
// Restated by oracle/transformer.py:rope_inv_freq and pinned against HF in
// tests/test_oracle_hf_pin.py.
void rope_inv_freq(float theta, float* inv64) {
  for (int i = 0; i < 64; ++i) {
    const float e = static_cast<float>(2 * i) / 128.0f;
    const float a = static_cast<float>(std::pow(static_cast<double>(theta), static_cast<double>(e)));
    inv64[i] = 1.0f / a;
  }
}

void set_rope_inv_freq(const float* inv_freq64, cudaStream_t s) {
  MRSP_CUDA(cudaMemcpyToSymbolAsync(c_inv_freq, inv_freq64, 64 * sizeof(float), 0,
                                    cudaMemcpyHostToDevice, s));
}

void rope(__nv_bfloat16* qkv, int ld, int col0, int n_heads, const int* pos, int n,
          cudaStream_t s) {
  if (n <= 0 || n_heads <= 0) return;
  MRSP_REQUIRE(ld % 2 == 0 && col0 % 2 == 0, MRSP_INVALID_ARGUMENT, "rope: odd leading dim");
  const int work = n * 32;
  launch_pdl(rope_kernel, dim3((work + 255) / 256), dim3(256), 0, s, qkv, ld, col0, n_heads, pos,
             n);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

void patchify(const float* pix, __nv_bfloat16* out, int F, int H, int W, int P, int kpad,
              cudaStream_t s) {
  const size_t total = static_cast<size_t>(F) * (H / P) * (W / P) * kpad;
  if (!total) return;
  MRSP_REQUIRE(kpad % 2 == 0 && kpad >= 3 * P * P, MRSP_INVALID_ARGUMENT, "patchify: bad kpad");
  const size_t smem = (static_cast<size_t>(3) * P * W + kpad) * sizeof(float);
  MRSP_REQUIRE(smem <= 200 * 1024, MRSP_INVALID_ARGUMENT, "patchify: image rows too wide");
  static const bool attr = [] {  // thread-safe one-time setup
    MRSP_CUDA(cudaFuncSetAttribute(patchify_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   200 * 1024));
    return true;
  }();
  (void)attr;
  patchify_kernel<<<F * (H / P), 256, smem, s>>>(pix, out, F, H, W, P, kpad);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

void broadcast_rows(const float* src, float* dst, int n, int period, int d, cudaStream_t s) {
  MRSP_REQUIRE(d % 4 == 0, MRSP_INVALID_ARGUMENT, "broadcast_rows: d % 4");
  const size_t total = static_cast<size_t>(n) * d / 4;
  if (!total) return;
  broadcast_rows_kernel<<<grid_for(total, 256), 256, 0, s>>>(src, dst, n, period, d);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

void pack_sequence(const __nv_bfloat16* frame_emb, int n_frame_tok, const int* question, int n_q,
                   const int* resp, const int* lengths, int Lmax, const __nv_bfloat16* embed,
                   int d, long p0, int n, float* hidden, int* pos_ids, unsigned char* pad_mask,
                   int* tok_out, cudaStream_t s) {
  if (n <= 0) return;
  MRSP_REQUIRE(d % 2 == 0, MRSP_INVALID_ARGUMENT, "pack: d % 2");
  pack_kernel<<<std::min(n, 148 * 8), 256, 0, s>>>(frame_emb, n_frame_tok, question, n_q, resp,
                                                   lengths, Lmax, embed, d, p0, n, hidden, pos_ids,
                                                   pad_mask, tok_out);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

void logprob_combine(const float2* part, int n_tiles, const float* tgt_logit, int n, float* lp,
                     float* lse, cudaStream_t s) {
  if (n <= 0) return;
  logprob_combine_kernel<<<(n + 7) / 8, 256, 0, s>>>(part, n_tiles, tgt_logit, n, lp, lse);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

void init_uniform_bf16(__nv_bfloat16* w, size_t n, uint64_t key, float scale, cudaStream_t s) {
  if (!n) return;
  init_uniform_bf16_kernel<<<grid_for(n, 256), 256, 0, s>>>(w, n, key, scale);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

void init_uniform_f32(float* w, size_t n, uint64_t key, float scale, float offset, cudaStream_t s) {
  if (!n) return;
  init_uniform_f32_kernel<<<grid_for(n, 256), 256, 0, s>>>(w, n, key, scale, offset);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

void convert_bf16_f32(const __nv_bfloat16* in, float* out, size_t n, cudaStream_t s) {
  if (!n) return;
  convert_bf16_f32_kernel<<<grid_for(n, 256), 256, 0, s>>>(in, out, n);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

}  // namespace mrsp
