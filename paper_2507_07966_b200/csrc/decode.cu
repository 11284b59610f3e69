// decode.cu — the kernels of rollout generation: decode
// attention over the cached prompt prefix + each row's own generated keys,
// the split merge, and temperature sampling with the old log-prob.
//
// Decode attention (one generation step, G rows): per kv head, the q_per_kv x G
// queries (<= 64) attend to the shared prefix K/V (computed once by the prefix
// prefill, [Lp][kv][128] per layer) and to the keys of their own row generated
// so far (time-major row cache [t][G][kv][128], row mask). The key range is
// split into chunks of DEC_CHUNK keys, one CTA per (chunk, kv head): each K/V
// tile read from HBM serves all of the kv group's queries (GQA reuse), and the
// CTA emits an unnormalised partial (m, l, O) merged by dec_merge_kernel —
// flash-decoding. Work per key is q·k and p·v for <= 64 queries (a few
// thousand FMAs per 256 B of K and V): CUDA-core FP32 is enough to keep the
// kernel near the HBM rate of the prefix KV stream.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "common.h"
#include "misc.h"

namespace mrsp {
namespace {

constexpr int DEC_QN = 64;      // max queries per kv head (q_per_kv x G)
constexpr int DEC_KT = 64;      // keys per smem tile
constexpr int DEC_CHUNK = 1024; // keys per CTA
constexpr int HD = 128;

struct DecArgs {
  const __nv_bfloat16* q;  // [G][ldq] bf16, head h at column q_col0 + 128 h
  int ldq, q_col0;
  const __nv_bfloat16* kv_prefix;  // [Lp][ld_kv]: K of kv head j at 128 j, V at v_off + 128 j
  const __nv_bfloat16* kv_rows;    // [(t+1) * G][ld_kv] time-major: row (s*G + g)
  int ld_kv, v_off;
  int Lp, G, t, q_per_kv, n_kv;
  int n_prefix_chunks, n_row_chunks;
  float scale_log2;
  float* part;  // [n_chunks][n_kv][DEC_QN][HD + 2]
};

__global__ void __launch_bounds__(256)
    dec_attn_kernel(DecArgs a) {
  extern __shared__ float sm[];
  float* Qs = sm;                          // [DEC_QN][HD]
  float* Ks = Qs + DEC_QN * HD;            // [DEC_KT][HD + 1]
  float* Vs = Ks + DEC_KT * (HD + 1);      // [DEC_KT][HD]
  float* Ps = Vs + DEC_KT * HD;            // [DEC_QN][DEC_KT + 1]
  const int chunk = blockIdx.x, kvh = blockIdx.y, tid = threadIdx.x;
  const int qn = a.q_per_kv * a.G;
  const bool rows_src = chunk >= a.n_prefix_chunks;
  const long k_begin = static_cast<long>(rows_src ? chunk - a.n_prefix_chunks : chunk) * DEC_CHUNK;
  const long k_total = rows_src ? static_cast<long>(a.t + 1) * a.G : a.Lp;
  const long k_end = std::min<long>(k_begin + DEC_CHUNK, k_total);
  const __nv_bfloat16* src = rows_src ? a.kv_rows : a.kv_prefix;
  // queries: index qi = hl * G + g (hl: head within the kv group)
  for (int i = tid; i < DEC_QN * HD; i += blockDim.x) {
    const int qi = i / HD, d = i % HD;
    float v = 0.f;
    if (qi < qn) {
      const int hl = qi / a.G, g = qi % a.G;
      v = __bfloat162float(a.q[static_cast<size_t>(g) * a.ldq + a.q_col0 +
                               (kvh * a.q_per_kv + hl) * HD + d]);
    }
    Qs[i] = v;
  }
  // thread -> (query, 16 keys) for S, (query, 32 head dims) for O
  const int q = tid >> 2, sub = tid & 3;
  const int g_of_q = q % max(a.G, 1);
  float m = -INFINITY, l = 0.f, o[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) o[j] = 0.f;
  for (long k0 = k_begin; k0 < k_end; k0 += DEC_KT) {
    __syncthreads();
    for (int i = tid; i < DEC_KT * (HD / 8); i += blockDim.x) {  // 16-byte loads
      const int kk = i / (HD / 8), c8 = (i % (HD / 8)) * 8;
      const long k = k0 + kk;
      float kv[8] = {0, 0, 0, 0, 0, 0, 0, 0}, vv[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      if (k < k_end) {
        const __nv_bfloat16* row = src + static_cast<size_t>(k) * a.ld_kv;
        const uint4 ku = *reinterpret_cast<const uint4*>(row + kvh * HD + c8);
        const uint4 vu = *reinterpret_cast<const uint4*>(row + a.v_off + kvh * HD + c8);
        const __nv_bfloat162* k2 = reinterpret_cast<const __nv_bfloat162*>(&ku);
        const __nv_bfloat162* v2 = reinterpret_cast<const __nv_bfloat162*>(&vu);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 kf = __bfloat1622float2(k2[e]), vf = __bfloat1622float2(v2[e]);
          kv[2 * e] = kf.x;
          kv[2 * e + 1] = kf.y;
          vv[2 * e] = vf.x;
          vv[2 * e + 1] = vf.y;
        }
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        Ks[kk * (HD + 1) + c8 + e] = kv[e];
        Vs[kk * HD + c8 + e] = vv[e];
      }
    }
    __syncthreads();
    // scores for 16 keys of this thread's query (log2 domain)
    float s[16];
    float mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int kk = sub * 16 + j;
      const long k = k0 + kk;
      float acc = 0.f;
#pragma unroll 8
      for (int d = 0; d < HD; ++d) acc = fmaf(Qs[q * HD + d], Ks[kk * (HD + 1) + d], acc);
      bool vis = q < qn && k < k_end;
      if (rows_src) vis = vis && static_cast<int>(k % a.G) == g_of_q;  // own row only
      s[j] = vis ? acc * a.scale_log2 : -INFINITY;
      mx = fmaxf(mx, s[j]);
    }
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    const float m_new = fmaxf(m, mx);
    const float alpha = m_new == -INFINITY ? 1.f : exp2f(m - m_new);
    float ls = 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float p = m_new == -INFINITY ? 0.f : exp2f(s[j] - m_new);
      Ps[q * (DEC_KT + 1) + sub * 16 + j] = p;
      ls += p;
    }
    ls += __shfl_xor_sync(0xffffffffu, ls, 1);
    ls += __shfl_xor_sync(0xffffffffu, ls, 2);
    l = l * alpha + ls;
    m = m_new;
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 32; ++j) o[j] *= alpha;
    for (int kk = 0; kk < DEC_KT; ++kk) {
      const float p = Ps[q * (DEC_KT + 1) + kk];
#pragma unroll
      for (int j = 0; j < 32; ++j) o[j] = fmaf(p, Vs[kk * HD + sub * 32 + j], o[j]);
    }
  }
  if (q < qn) {
    float* out = a.part + ((static_cast<size_t>(chunk) * a.n_kv + kvh) * DEC_QN + q) * (HD + 2);
#pragma unroll
    for (int j = 0; j < 32; ++j) out[sub * 32 + j] = o[j];
    if (sub == 0) {
      out[HD] = m;
      out[HD + 1] = l;
    }
  }
}

// O[g][h*128 + d] = sum_c O_c 2^(m_c - m) / sum_c l_c 2^(m_c - m)
__global__ void dec_merge_kernel(const float* __restrict__ part, int n_chunks, int n_kv,
                                 int q_per_kv, int G, __nv_bfloat16* __restrict__ out, int ldo) {
  const int qi = blockIdx.x, kvh = blockIdx.y, d = threadIdx.x;  // blockDim = 128
  const int hl = qi / G, g = qi % G;
  float m = -INFINITY;
  for (int c = 0; c < n_chunks; ++c)
    m = fmaxf(m, part[((static_cast<size_t>(c) * n_kv + kvh) * DEC_QN + qi) * (HD + 2) + HD]);
  float l = 0.f, o = 0.f;
  for (int c = 0; c < n_chunks; ++c) {
    const float* p = part + ((static_cast<size_t>(c) * n_kv + kvh) * DEC_QN + qi) * (HD + 2);
    if (p[HD] == -INFINITY) continue;
    const float w = exp2f(p[HD] - m);
    l += p[HD + 1] * w;
    o += p[d] * w;
  }
  out[static_cast<size_t>(g) * ldo + (kvh * q_per_kv + hl) * HD + d] =
      __float2bfloat16_rn(l > 0.f ? o / l : 0.f);
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// One CTA per row: p = softmax(logits / T); token = first v with cdf(v) > u,
// u = (splitmix64(seed, row, t) >> 11) * 2^-53; old_lp = log_softmax(logits)[token]
// at temperature 1 (policy.cpp:130-134). Rows already finished (EOS) only
// record PAD. One thread-block scan over the vocabulary, fp64 accumulation.
__global__ void __launch_bounds__(1024)
    sample_kernel(const float* __restrict__ logits, int V, float inv_temp, uint64_t seed, int t,
                  int* __restrict__ done, int* __restrict__ tokens, float* __restrict__ old_lp,
                  int* __restrict__ lengths, int max_len, int eos, int pad) {
  const int g = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  __shared__ double red[32];
  __shared__ float redf[32];
  __shared__ int pick;
  if (done[g]) {
    if (tid == 0) tokens[static_cast<size_t>(g) * max_len + t] = pad;
    return;
  }
  const float* x = logits + static_cast<size_t>(g) * V;
  auto block_max = [&](float v) {
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((tid & 31) == 0) redf[tid >> 5] = v;
    __syncthreads();
    if (tid < 32) {
      v = tid < (nt >> 5) ? redf[tid] : -INFINITY;
      for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
      if (tid == 0) redf[0] = v;
    }
    __syncthreads();
    const float r = redf[0];
    __syncthreads();
    return r;
  };
  auto block_sum = [&](double v) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((tid & 31) == 0) red[tid >> 5] = v;
    __syncthreads();
    if (tid < 32) {
      v = tid < (nt >> 5) ? red[tid] : 0.0;
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (tid == 0) red[0] = v;
    }
    __syncthreads();
    const double r = red[0];
    __syncthreads();
    return r;
  };
  float mx = -INFINITY;
  for (int v = tid; v < V; v += nt) mx = fmaxf(mx, x[v]);
  mx = block_max(mx);
  double zs = 0.0, z1 = 0.0;  // sum exp((x - mx) / T), sum exp(x - mx)
  for (int v = tid; v < V; v += nt) {
    zs += exp((static_cast<double>(x[v]) - mx) * inv_temp);
    z1 += exp(static_cast<double>(x[v]) - mx);
  }
  zs = block_sum(zs);
  z1 = block_sum(z1);
  const double u = static_cast<double>(mix64(seed ^ mix64((static_cast<uint64_t>(g) << 32) |
                                                         static_cast<uint32_t>(t))) >> 11) *
                   0x1.0p-53 * zs;
  // inverse CDF: each thread owns a contiguous slice; exclusive scan of the
  // slice sums finds the slice containing u, then that thread walks it
  const int per = (V + nt - 1) / nt, v0 = tid * per, v1 = min(V, v0 + per);
  double mine = 0.0;
  for (int v = v0; v < v1; ++v) mine += exp((static_cast<double>(x[v]) - mx) * inv_temp);
  // block-wide inclusive scan via warp scans
  double inc = mine;
  for (int o = 1; o < 32; o <<= 1) {
    const double n = __shfl_up_sync(0xffffffffu, inc, o);
    if ((tid & 31) >= o) inc += n;
  }
  if ((tid & 31) == 31) red[tid >> 5] = inc;
  if (tid == 0) pick = V - 1;
  __syncthreads();
  if (tid < 32) {
    double w = tid < (nt >> 5) ? red[tid] : 0.0;
    for (int o = 1; o < 32; o <<= 1) {
      const double n = __shfl_up_sync(0xffffffffu, w, o);
      if (tid >= o) w += n;
    }
    red[tid] = w;  // inclusive over warps
  }
  __syncthreads();
  const double before = inc - mine + ((tid >> 5) ? red[(tid >> 5) - 1] : 0.0);
  if (u >= before && u < before + mine) {
    double c = before;
    int chosen = v1 - 1;
    for (int v = v0; v < v1; ++v) {
      c += exp((static_cast<double>(x[v]) - mx) * inv_temp);
      if (u < c) {
        chosen = v;
        break;
      }
    }
    pick = chosen;
  }
  __syncthreads();
  if (tid == 0) {
    const int tok = pick;
    tokens[static_cast<size_t>(g) * max_len + t] = tok;
    old_lp[static_cast<size_t>(g) * max_len + t] =
        static_cast<float>(static_cast<double>(x[tok]) - mx - log(z1));
    lengths[g] = t + 1;
    if (tok == eos) done[g] = 1;
  }
}

// hidden[g] = embed[prev token of row g] (EOS at t = 0, policy.cpp:127), and
// the position id Lp + t of every row (rows restart at Lp, as in the pack).
__global__ void decode_embed_kernel(const __nv_bfloat16* __restrict__ embed, int d,
                                    const int* __restrict__ tokens, int max_len, int t, int pos,
                                    float* __restrict__ hidden, int* __restrict__ pos_out) {
  const int g = blockIdx.x;
  const int tok = t == 0 ? 1 /* Vocab::kEos */ : tokens[static_cast<size_t>(g) * max_len + t - 1];
  if (threadIdx.x == 0) pos_out[g] = pos;
  const __nv_bfloat162* src = reinterpret_cast<const __nv_bfloat162*>(embed + static_cast<size_t>(tok) * d);
  float2* dst = reinterpret_cast<float2*>(hidden + static_cast<size_t>(g) * d);
  for (int i = threadIdx.x; i < d / 2; i += blockDim.x) dst[i] = __bfloat1622float2(src[i]);
}

}  // namespace

void decode_embed(const __nv_bfloat16* embed, int d, const int* tokens, int max_len, int t, int G,
                  int pos, float* hidden, int* pos_out, cudaStream_t s) {
  decode_embed_kernel<<<G, 256, 0, s>>>(embed, d, tokens, max_len, t, pos, hidden, pos_out);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

size_t decode_partial_bytes(int max_prefix, int max_len, int G, int n_kv) {
  const int chunks = (max_prefix + DEC_CHUNK - 1) / DEC_CHUNK +
                     (max_len * G + DEC_CHUNK - 1) / DEC_CHUNK;
  return static_cast<size_t>(chunks) * n_kv * DEC_QN * (HD + 2) * sizeof(float);
}

void decode_attention(const void* q, int ldq, int q_col0, const void* kv_prefix,
                      const void* kv_rows, int ld_kv, int v_off, int Lp, int G, int t,
                      int q_per_kv, int n_kv, float scale, float* part, void* out, int ldo,
                      cudaStream_t s) {
  MRSP_REQUIRE(q_per_kv * G <= DEC_QN, MRSP_INVALID_ARGUMENT,
               "generate: q_per_kv x G must be <= 64");
  DecArgs a;
  a.q = static_cast<const __nv_bfloat16*>(q);
  a.ldq = ldq;
  a.q_col0 = q_col0;
  a.kv_prefix = static_cast<const __nv_bfloat16*>(kv_prefix);
  a.kv_rows = static_cast<const __nv_bfloat16*>(kv_rows);
  a.ld_kv = ld_kv;
  a.v_off = v_off;
  a.Lp = Lp;
  a.G = G;
  a.t = t;
  a.q_per_kv = q_per_kv;
  a.n_kv = n_kv;
  a.n_prefix_chunks = (Lp + DEC_CHUNK - 1) / DEC_CHUNK;
  a.n_row_chunks = ((t + 1) * G + DEC_CHUNK - 1) / DEC_CHUNK;
  a.scale_log2 = scale * 1.4426950408889634f;
  a.part = part;
  const size_t smem =
      (DEC_QN * HD + DEC_KT * (HD + 1) + DEC_KT * HD + DEC_QN * (DEC_KT + 1)) * sizeof(float);
  static const bool attr = [smem] {
    MRSP_CUDA(cudaFuncSetAttribute(dec_attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
    return true;
  }();
  (void)attr;
  const int chunks = a.n_prefix_chunks + a.n_row_chunks;
  dec_attn_kernel<<<dim3(chunks, n_kv), 256, smem, s>>>(a);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
  dec_merge_kernel<<<dim3(q_per_kv * G, n_kv), HD, 0, s>>>(part, chunks, n_kv, q_per_kv, G,
                                                           static_cast<__nv_bfloat16*>(out), ldo);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

void sample_tokens(const float* logits, int G, int V, float temperature, uint64_t seed, int t,
                   int* done, int* tokens, float* old_lp, int* lengths, int max_len,
                   cudaStream_t s) {
  sample_kernel<<<G, 1024, 0, s>>>(logits, V, 1.0f / temperature, seed, t, done, tokens, old_lp,
                                   lengths, max_len, /*Vocab::kEos*/ 1, /*Vocab::kPad*/ 0);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

}  // namespace mrsp
