// gemm.cu — persistent, warp-specialised tcgen05 BF16 GEMM for sm_100a.
//
//   C[M,N] = epilogue( A[M,K] . B[N,K]^T )      A, B bf16 K-major, fp32 accumulate
//
// Default kernel: single CTA, 128 x 256 tiles (a CTA-pair variant,
// gemm_bf16_pair below, is selectable with MRSP_GEMM_IMPL; see kDefaultGemmImpl):
//   warp 0      TMA producer: A/B 128x64 / 256x64 tiles -> 4-stage smem ring
//   warp 1      MMA issuer: one elected lane issues tcgen05.mma 128x256x16 into
//               a double-buffered TMEM accumulator (2 x 256 fp32 columns)
//   warp 2      TMEM allocator
//   warps 4-7   epilogue: tcgen05.ld 32x32b -> registers -> fused op -> global
// The epilogue of tile i overlaps the MMA of tile i+1 (TMEM double buffer).
// Smem descriptors are SWIZZLE_128B K-major, matching the TMA tensor maps.
//
// Fused epilogues (the LLM / vision layers' elementwise tails, so no separate
// HBM pass): +bias, +bias then GELU(tanh), SwiGLU over [gate|up] N-halves,
// fp32 residual accumulate (hidden += A.B^T [+ bias]), plain bf16 / fp32 store,
// LM-head log-prob partials.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "common.h"
#include "gemm.h"
#include "misc.h"
#include "pdl.cuh"
#include "rownorm.cuh"
#include "sm100.cuh"
#include "tma.h"

namespace mrsp {
namespace {

using namespace sm100;

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int TMEM_COLS = 512;  // two 128x256 fp32 accumulators
constexpr int THREADS = 256;
// Staged epilogue: per epilogue warp two 32-row x 128-byte boxes (SW128) that
// TMA stores (or reduce-adds) to global while the next box is being filled.
constexpr int OUT_BOX = 32 * 128;
constexpr int OUT_BYTES = 4 * 2 * OUT_BOX;
constexpr size_t SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + OUT_BYTES + 256;

struct EpiArgs {
  int M, N, K;
  int epi;
  int vec_ok;  // output/residual rows are 16-byte aligned -> vector stores
  int staged;  // epilogue goes through smem + TMA store / reduce-add (tmC)
  int k_splits;  // > 1: fp32 partials of K range ks to ws[ks][M][N]
  float* ws;
  void* C;
  int ldc;
  const float* bias;
  float* resid;
  int ldr;
  const int* targets;  // LOGPROB: target id per row
  float2* part;        // LOGPROB: [M][n_tiles] (tile max, sum exp(x - max))
  float* tgt_logit;    // LOGPROB: logit of the target per row
  // QKV_SCATTER (see GemmArgs)
  const int* pos;
  const float* inv_freq;
  int n_rope_blocks;
  long row0;
  const int2* route;
  void* const* peer_base;
  const int* peer_ld;
  int row_blocks;
  // decode fusions of the split-K reduction (GemmArgs::post)
  int post;
  __nv_bfloat16* kv_rows;
  int kvw, kv_col0;
  const int* tdev;
  const float* norm_w;
  __nv_bfloat16* norm_out;
  int ld_norm;
  float norm_eps;
  // GEMM_EPI_SWIGLU_BWD (GemmArgs::aux / aux_out)
  const __nv_bfloat16* aux;
  int ld_aux;
  __nv_bfloat16* aux_out;
  int ld_aux_out;
};

// Grouped raster: consecutive tiles sweep a GROUP_M-tall band of m-tiles with
// n varying slowest inside the band, so the ~148 concurrently running tiles
// touch ~16 A-tiles and ~10 B-tiles instead of 1 A-row against all of B.
constexpr int GROUP_M = 16;
__device__ __forceinline__ void tile_coords(int tile, int m_tiles, int n_tiles, int& mt, int& nt) {
  const int band = tile / (GROUP_M * n_tiles);
  const int first_m = band * GROUP_M;
  const int rows = min(GROUP_M, m_tiles - first_m);
  const int local = tile - band * GROUP_M * n_tiles;
  mt = first_m + local % rows;
  nt = local / rows;
}

// Epilogue activations on the SFU (MUFU.TANH / MUFU.EX2 + fast reciprocal):
// the outputs are rounded to bf16 (rel. 2^-9), far coarser than the
// approximations' ~2^-11; an IEEE division per element made the SwiGLU
// epilogue slower than the 128x256x3584 main loop it overlaps.
__device__ __forceinline__ float tanh_fast(float x) {
#ifdef MRSP_NUMERICS_PROBE_ACCURATE_TANH  // numerics probe builds only (tools/vision_numerics.py)
  return tanhf(x);
#endif
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float gelu_tanh(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  return 0.5f * x * (1.0f + tanh_fast(k0 * (x + k1 * x * x * x)));
}
__device__ __forceinline__ float silu(float x) { return __fdividef(x, 1.0f + __expf(-x)); }

// Fused epilogue of one accumulator tile row slice: TMEM row `t_row` (this
// thread's lane, BN fp32 columns) -> the epilogue op -> global. Shared by the
// single-CTA and the CTA-pair kernels.
template <int kBN = BN>
__device__ __forceinline__ void epilogue_row(const EpiArgs& args, uint32_t t_row, int row,
                                             bool row_ok, int nt, int n_tiles) {
  if (args.epi == GEMM_EPI_QKV_SCATTER) {
    // Fused Ulysses sequence -> head all-to-all: this tile's two 128-column
    // head blocks get +bias, bf16 rounding and (q, k heads) rotate-half RoPE
    // exactly as the BIAS_BF16 epilogue followed by the rope kernel would
    // compute them, then go straight to the owner rank's head-shard buffer
    // (a peer GPU's memory over NVLink, or a virtual rank's buffer).
    const float p = row_ok ? static_cast<float>(args.pos[row]) : 0.f;
    const long grow = args.row0 + row;
#pragma unroll 1
    for (int hl = 0; hl < kBN / 128; ++hl) {
      const int hb = nt * (kBN / 128) + hl;
      if (hb * 128 >= args.N) break;  // warp-uniform
      const bool rope = hb < args.n_rope_blocks;
      const int2 d0 = args.route[2 * hb], d1 = args.route[2 * hb + 1];
#pragma unroll 1
      for (int j = 0; j < 64; j += 32) {
        uint32_t ra[32], rb[32];
        tmem_ld32(t_row + hl * 128 + j, ra);
        tmem_ld32(t_row + hl * 128 + 64 + j, rb);
        tmem_ld_wait();
        if (row_ok) {
          uint32_t oa[16], ob[16];
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            float x1[2], x2[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int c = hb * 128 + j + i + e;
              x1[e] = __bfloat162float(__float2bfloat16_rn(__uint_as_float(ra[i + e]) + args.bias[c]));
              x2[e] = __bfloat162float(__float2bfloat16_rn(__uint_as_float(rb[i + e]) + args.bias[c + 64]));
              if (rope) {
                float sn, cs;
                sincosf(__fmul_rn(p, args.inv_freq[j + i + e]), &sn, &cs);
                const float y1 = __fsub_rn(__fmul_rn(x1[e], cs), __fmul_rn(x2[e], sn));
                const float y2 = __fadd_rn(__fmul_rn(x2[e], cs), __fmul_rn(x1[e], sn));
                x1[e] = y1;
                x2[e] = y2;
              }
            }
            oa[i / 2] = pack_bf16(x1[0], x1[1]);
            ob[i / 2] = pack_bf16(x2[0], x2[1]);
          }
          // destinations: d0 and d1 (x < 0: none); d1 = (-2, m): ONE of the m
          // ranks from d0.x, by the row's query block (query-row split); d1 =
          // (-3, m): all m ranks from d0.x (the shared K / V head)
          const int n_to = d1.x == -3 ? d1.y : d1.x == -2 ? 1 : 2;
#pragma unroll 1
          for (int t = 0; t < n_to; ++t) {
            int2 dd = t ? d1 : d0;
            if (d1.x == -2)
              dd = make_int2(d0.x + attn_row_part(static_cast<int>(grow / ATTN_ROW_BLOCK),
                                                  args.row_blocks, d1.y), d0.y);
            else if (d1.x == -3)
              dd = make_int2(d0.x + t, d0.y);
            if (dd.x < 0) continue;
            __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(args.peer_base[dd.x]) +
                                 grow * args.peer_ld[dd.x] + dd.y + j;
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
              reinterpret_cast<uint4*>(dst)[q4] =
                  make_uint4(oa[4 * q4], oa[4 * q4 + 1], oa[4 * q4 + 2], oa[4 * q4 + 3]);
              reinterpret_cast<uint4*>(dst + 64)[q4] =
                  make_uint4(ob[4 * q4], ob[4 * q4 + 1], ob[4 * q4 + 2], ob[4 * q4 + 3]);
            }
          }
        }
      }
    }
  } else if (args.epi == GEMM_EPI_LOGPROB_PARTIAL) {
    // Fused vocabulary projection + log-softmax pieces: this 256-wide vocab
    // tile's (max, sum exp) per row and the target logit if it lies here.
    // Logits never leave TMEM/registers.
    const int tgt = row_ok ? args.targets[row] : -1;
    float m = -INFINITY, ssum = 0.f;
    for (int c = 0; c < kBN; c += 32) {
      uint32_t r[32];
      tmem_ld32(t_row + c, r);
      tmem_ld_wait();
      const int col = nt * kBN + c;
      float cm = -INFINITY;
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (col + j < args.N) cm = fmaxf(cm, __uint_as_float(r[j]));
      const float mn = fmaxf(m, cm);
      float acc_s = (m == -INFINITY) ? 0.f : ssum * __expf(m - mn);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float x = __uint_as_float(r[j]);
        if (col + j < args.N) acc_s += __expf(x - mn);
        if (col + j == tgt) args.tgt_logit[row] = x;
      }
      m = mn;
      ssum = acc_s;
    }
    if (row_ok) args.part[static_cast<size_t>(row) * n_tiles + nt] = make_float2(m, ssum);
  } else if (args.epi == GEMM_EPI_SWIGLU_BWD) {
    // SwiGLU backward: with s = sigmoid(g), silu(g) = g s, silu'(g) = s (1 + g (1 - s)),
    //   dg = dA u silu'(g), du = dA silu(g)   -> C[:, nt*256 + j] | C[:, nt*256 + 128 + j]
    // and the forward output silu(g) u (bit-identical to GEMM_EPI_SWIGLU_BF16) -> aux_out
    __nv_bfloat16* C = static_cast<__nv_bfloat16*>(args.C);
    for (int c = 0; c < kBN / 2; c += 32) {
      uint32_t g[32], u[32];
      tmem_ld32(t_row + c, g);
      tmem_ld32(t_row + kBN / 2 + c, u);
      tmem_ld_wait();
      const int col = nt * (kBN / 2) + c;
      if (row_ok) {
        const uint4* da4 = reinterpret_cast<const uint4*>(args.aux + static_cast<size_t>(row) * args.ld_aux + col);
        uint32_t dar[16];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint4 v = da4[j];
          dar[4 * j] = v.x; dar[4 * j + 1] = v.y; dar[4 * j + 2] = v.z; dar[4 * j + 3] = v.w;
        }
        uint32_t og[16], ou[16], oa[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float2 da = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&dar[j]));
          float rg[2], ru[2], ra[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const float gv = __uint_as_float(g[2 * j + e]), uv = __uint_as_float(u[2 * j + e]);
            const float dv = e ? da.y : da.x;
            const float sg = __fdividef(1.0f, 1.0f + __expf(-gv));
            const float sl = silu(gv);
            rg[e] = dv * uv * (sg * (1.0f + gv * (1.0f - sg)));
            ru[e] = dv * sl;
            ra[e] = sl * uv;
          }
          og[j] = pack_bf16(rg[0], rg[1]);
          ou[j] = pack_bf16(ru[0], ru[1]);
          oa[j] = pack_bf16(ra[0], ra[1]);
        }
        uint4* dg = reinterpret_cast<uint4*>(C + static_cast<size_t>(row) * args.ldc + nt * kBN + c);
        uint4* du = reinterpret_cast<uint4*>(C + static_cast<size_t>(row) * args.ldc + nt * kBN + kBN / 2 + c);
        uint4* ac = reinterpret_cast<uint4*>(args.aux_out + static_cast<size_t>(row) * args.ld_aux_out + col);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          dg[j] = make_uint4(og[4 * j], og[4 * j + 1], og[4 * j + 2], og[4 * j + 3]);
          du[j] = make_uint4(ou[4 * j], ou[4 * j + 1], ou[4 * j + 2], ou[4 * j + 3]);
          ac[j] = make_uint4(oa[4 * j], oa[4 * j + 1], oa[4 * j + 2], oa[4 * j + 3]);
        }
      }
    }
  } else if (args.epi == GEMM_EPI_SWIGLU_BF16) {
    // columns [0,128) are gate, [128,256) the matching up projections
    __nv_bfloat16* C = static_cast<__nv_bfloat16*>(args.C);
    for (int c = 0; c < kBN / 2; c += 32) {
      uint32_t g[32], u[32];
      tmem_ld32(t_row + c, g);
      tmem_ld32(t_row + kBN / 2 + c, u);
      tmem_ld_wait();
      const int col = nt * (kBN / 2) + c;
      if (row_ok) {
        uint32_t o[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float a0 = silu(__uint_as_float(g[2 * j])) * __uint_as_float(u[2 * j]);
          const float a1 = silu(__uint_as_float(g[2 * j + 1])) * __uint_as_float(u[2 * j + 1]);
          o[j] = pack_bf16(a0, a1);
        }
        uint4* dst = reinterpret_cast<uint4*>(C + static_cast<size_t>(row) * args.ldc + col);
        if (args.vec_ok && col + 32 <= args.N / 2) {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            dst[j] = make_uint4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
        } else {
          const __nv_bfloat16* ob = reinterpret_cast<const __nv_bfloat16*>(o);
          for (int j = 0; j < 32 && col + j < args.N / 2; ++j)
            C[static_cast<size_t>(row) * args.ldc + col + j] = ob[j];
        }
      }
    }
  } else {
    for (int c = 0; c < kBN; c += 32) {
      uint32_t r[32];
      tmem_ld32(t_row + c, r);
      tmem_ld_wait();
      const int col = nt * kBN + c;
      if (row_ok && col < args.N) {  // stores only; the TMEM load above is warp-wide
      float v[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
      const bool full_chunk = col + 32 <= args.N;
      const bool vec = full_chunk && args.vec_ok;
      if (args.bias) {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (full_chunk || col + j < args.N) v[j] += args.bias[col + j];
      }
      if (args.epi == GEMM_EPI_BIAS_GELU_BF16) {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = gelu_tanh(v[j]);
      }
      if (args.epi == GEMM_EPI_RESID_F32) {
        float* R = args.resid + static_cast<size_t>(row) * args.ldr + col;
        if (vec) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float4 x = reinterpret_cast<float4*>(R)[j];
            x.x += v[4 * j]; x.y += v[4 * j + 1]; x.z += v[4 * j + 2]; x.w += v[4 * j + 3];
            reinterpret_cast<float4*>(R)[j] = x;
          }
        } else {
          for (int j = 0; j < 32 && col + j < args.N; ++j) R[j] += v[j];
        }
      } else if (args.epi == GEMM_EPI_STORE_F32) {
        float* Cf = static_cast<float*>(args.C) + static_cast<size_t>(row) * args.ldc + col;
        if (vec) {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            reinterpret_cast<float4*>(Cf)[j] =
                make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        } else {
          for (int j = 0; j < 32 && col + j < args.N; ++j) Cf[j] = v[j];
        }
      } else {  // bf16 stores: STORE / BIAS / BIAS_GELU
        __nv_bfloat16* Cb =
            static_cast<__nv_bfloat16*>(args.C) + static_cast<size_t>(row) * args.ldc + col;
        uint32_t o[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) o[j] = pack_bf16(v[2 * j], v[2 * j + 1]);
        if (vec) {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            reinterpret_cast<uint4*>(Cb)[j] =
                make_uint4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
        } else {
          const __nv_bfloat16* ob = reinterpret_cast<const __nv_bfloat16*>(o);
          for (int j = 0; j < 32 && col + j < args.N; ++j) Cb[j] = ob[j];
        }
      }
      }
    }
  }
}

// Uniform (warp-broadcast) bias loads for `n` columns starting at `col`;
// columns at or past N read as 0 (their outputs are clipped by the TMA store).
// No bias reads as -0, the additive identity (x + -0 == x, signed zeros kept).
template <int n>
__device__ __forceinline__ void load_bias(const float* bias, int col, int N, float (&b)[n]) {
  if (bias == nullptr) {
#pragma unroll
    for (int j = 0; j < n; ++j) b[j] = -0.f;
  } else if (col + n <= N) {
#pragma unroll
    for (int j = 0; j < n; j += 4) {
      const float4 x = __ldg(reinterpret_cast<const float4*>(bias + col + j));
      b[j] = x.x; b[j + 1] = x.y; b[j + 2] = x.z; b[j + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < n; ++j) b[j] = col + j < N ? bias[col + j] : 0.f;
  }
}

// Staged epilogue of one warp's 32 accumulator rows: per 128-byte output chunk
// (64 bf16 or 32 fp32 columns) TMEM -> registers -> fused op -> this warp's
// SW128 smem box (row = lane; 16-byte unit u of row r at u ^ (r & 7), so the
// row-per-lane st.shared are conflict-free) -> one TMA store (fp32 residual:
// TMA reduce-add in L2, i.e. resid += v rounded once, as the load/add/store
// path). Two boxes per warp: filling one overlaps the other's bulk copy.
// Rows past M / columns past N are clipped by the TMA unit.
template <int kBN = BN>
__device__ __forceinline__ void epilogue_staged(const EpiArgs& args, const CUtensorMap* tmC,
                                                uint32_t t_row, int y, int nt, uint8_t* boxes,
                                                uint32_t& buf) {
  const int lane = lane_id();
  const bool f32 = args.epi == GEMM_EPI_RESID_F32 || args.epi == GEMM_EPI_STORE_F32;
  const bool swiglu = args.epi == GEMM_EPI_SWIGLU_BF16;
  const int out_cols = swiglu ? kBN / 2 : kBN;
  const int col0 = nt * out_cols;
  const int out_n = swiglu ? args.N / 2 : args.N;
#pragma unroll 1
  for (int c = 0; c < out_cols; c += f32 ? 32 : 64) {
    if (col0 + c >= out_n) break;  // warp-uniform: the whole box is past N
    uint32_t w[32];  // this lane's 128 output bytes
    if (f32) {
      uint32_t r[32];
      tmem_ld32(t_row + c, r);
      float b[32];
      load_bias<32>(args.bias, col0 + c, args.N, b);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) w[j] = __float_as_uint(__uint_as_float(r[j]) + b[j]);
    } else if (swiglu) {
#pragma unroll
      for (int h = 0; h < 64; h += 32) {
        uint32_t g[32], u[32];
        tmem_ld32(t_row + c + h, g);
        tmem_ld32(t_row + kBN / 2 + c + h, u);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j)
          w[h / 2 + j] = pack_bf16(silu(__uint_as_float(g[2 * j])) * __uint_as_float(u[2 * j]),
                                   silu(__uint_as_float(g[2 * j + 1])) * __uint_as_float(u[2 * j + 1]));
      }
    } else {
      const bool gelu = args.epi == GEMM_EPI_BIAS_GELU_BF16;
#pragma unroll
      for (int h = 0; h < 64; h += 32) {
        uint32_t r[32];
        tmem_ld32(t_row + c + h, r);
        float b[32];
        load_bias<32>(args.bias, col0 + c + h, args.N, b);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          float v0 = __uint_as_float(r[2 * j]) + b[2 * j];
          float v1 = __uint_as_float(r[2 * j + 1]) + b[2 * j + 1];
          if (gelu) {
            v0 = gelu_tanh(v0);
            v1 = gelu_tanh(v1);
          }
          w[h / 2 + j] = pack_bf16(v0, v1);
        }
      }
    }
    uint8_t* box = boxes + buf * OUT_BOX;
    if (lane == 0) bulk_wait_read<1>();  // the copy that last read this box is done
    __syncwarp();
    const uint32_t row = smem_u32(box) + lane * 128;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      st_shared_v4(row + ((u ^ (lane & 7)) << 4), w[4 * u], w[4 * u + 1], w[4 * u + 2],
                   w[4 * u + 3]);
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      if (args.epi == GEMM_EPI_RESID_F32)
        tma_reduce_add_2d(tmC, smem_u32(box), col0 + c, y);
      else
        tma_store_2d(tmC, smem_u32(box), col0 + c, y);
      bulk_commit();
    }
    buf ^= 1;
  }
}

// kStages / kARows: the ring depth and the rows of A loaded per stage. The
// default (4, 128) serves every prefill GEMM. The skinny variant (6, 16) is for
// M <= 16 (the decode steps' G rows): each stage holds a 16-row A box (2 KB)
// in front of its 32 KB B tile, so 6 stages of weights are in flight instead of
// 4; the M = 128 MMA still reads 128 A rows, rows 16..127 being whatever bytes
// follow in the stage (the B tile) — they only produce accumulator rows >= 16,
// which no epilogue stores. No staged-epilogue boxes (row epilogue only).
template <int kStages, int kARows, int kBN = BN>
struct GemmCfg {
  static constexpr int kABytes = kARows * BK * 2;
  static constexpr int kBBytes = kBN * BK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kOutBytes = kARows == BM ? OUT_BYTES : 0;
  static constexpr size_t kSmem = 1024 + kStages * kStageBytes + kOutBytes + 256;
  static_assert(kABytes % 1024 == 0, "A box = whole SW128 atoms");
  static_assert(kARows == BM || kStageBytes >= A_BYTES, "MMA reads 128 A rows inside the stage");
};

// kMajor: bit 0 = A stored MN-major (A^T rows: element (m, k) at A[k * lda + m]),
// bit 1 = B stored MN-major (element (n, k) at B[k * ldb + n]) — the backward
// pass's dgrad (B = a weight read as its transpose) and wgrad (both operands
// token-major) GEMMs. An MN-major operand tile is loaded as 64 x 64 boxes
// (64 K rows x 128 bytes of M/N) and read through MN-major SW128 descriptors
// (LBO = one 64-wide box, 8 KB); the instruction descriptor's transpose bits
// tell the tensor core. kMajor 0 is the forward kernel, unchanged.
constexpr int MN_BOX = 64 * 64 * 2;
// kBN: output-tile width (256; 192 for N = 1152 / 3456-shaped GEMMs, where
// 256-wide tiles would leave a half-empty last tile).
template <int kStages, int kARows, int kMajor = 0, int kBN = BN>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_bf16_tcgen05(const __grid_constant__ CUtensorMap tmA,
                      const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ CUtensorMap tmC, EpiArgs args) {
  constexpr bool kAMN = (kMajor & 1) != 0, kBMN = (kMajor & 2) != 0;
  static_assert(kMajor == 0 || kARows == BM, "MN-major operands: full tiles only");
  using Cfg = GemmCfg<kStages, kARows, kBN>;
  constexpr int STAGES = kStages;
  constexpr int STAGE_BYTES = Cfg::kStageBytes;
  constexpr int A_STAGE = Cfg::kABytes;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* out_boxes = smem + STAGES * STAGE_BYTES;  // [4 warps][2][OUT_BOX] (default only)
  uint64_t* full = reinterpret_cast<uint64_t*>(out_boxes + Cfg::kOutBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;   // [2]
  uint64_t* tempty = tfull + 2;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = warp_id();
  const int m_tiles = (args.M + BM - 1) / BM;
  const int n_tiles = (args.N + kBN - 1) / kBN;
  const int ks_n = args.k_splits;
  const int num_tiles = m_tiles * n_tiles * ks_n;
  const int k_blocks = (args.K + BK - 1) / BK;
  // work item -> (m tile, n tile, K split [kb0, kb1))
  auto decode_tile = [&](int tile, int& mt, int& nt, int& kb0, int& kb1) {
    const int ks = tile % ks_n;
    tile_coords(tile / ks_n, m_tiles, n_tiles, mt, nt);
    kb0 = ks * k_blocks / ks_n;
    kb1 = (ks + 1) * k_blocks / ks_n;
  };

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (args.staged) tma_prefetch_desc(&tmC);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // Programmatic dependent launch (decode graphs): the successor may become
  // resident now; the weights (B) of the first stages do not depend on the
  // predecessor kernel, so the producer streams them in before pdl_wait() and
  // only the activation (A) loads and the epilogue's global accesses wait.
  // Without PDL both instructions are no-ops.
  pdl_trigger();

  auto load_a = [&](uint8_t* dst, uint64_t* bar, int kb, int mt) {
    if constexpr (kAMN) {
#pragma unroll
      for (int c = 0; c < BM / 64; ++c) tma_load_2d(dst + c * MN_BOX, &tmA, bar, mt * BM + c * 64, kb * BK);
    } else {
      tma_load_2d(dst, &tmA, bar, kb * BK, mt * BM);
    }
  };
  auto load_b = [&](uint8_t* dst, uint64_t* bar, int kb, int nt) {
    if constexpr (kBMN) {
#pragma unroll
      for (int c = 0; c < kBN / 64; ++c) tma_load_2d(dst + c * MN_BOX, &tmB, bar, nt * kBN + c * 64, kb * BK);
    } else {
      tma_load_2d(dst, &tmB, bar, kb * BK, nt * kBN);
    }
  };
  if (warp == 0) {
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      int pre = 0;  // first-tile k blocks whose B load was issued before the wait
      if (static_cast<int>(blockIdx.x) < num_tiles) {
        int mt, nt, kb0, kb1;
        decode_tile(blockIdx.x, mt, nt, kb0, kb1);
        for (; pre < STAGES && kb0 + pre < kb1; ++pre) {
          mbar_arrive_expect_tx(&full[pre], STAGE_BYTES);  // stages start empty
          load_b(smem + pre * STAGE_BYTES + A_STAGE, &full[pre], kb0 + pre, nt);
        }
      }
      pdl_wait();
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        int mt, nt, kb0, kb1;
        decode_tile(tile, mt, nt, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          uint8_t* sa = smem + stage * STAGE_BYTES;
          if (pre > 0 && tile == static_cast<int>(blockIdx.x) && kb - kb0 < pre) {
            load_a(sa, &full[stage], kb, mt);  // B already in flight
          } else {
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
            load_a(sa, &full[stage], kb, mt);
            load_b(sa + A_STAGE, &full[stage], kb, nt);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc =
        idesc_bf16_f32(BM, kBN) | (kAMN ? (1u << 15) : 0u) | (kBMN ? (1u << 16) : 0u);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      int mt, nt, kb0, kb1;
      decode_tile(tile, mt, nt, kb0, kb1);
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * kBN;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a_addr = smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t b_addr = a_addr + A_STAGE;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // K-major: the 16-element K step is 32 bytes along the row; MN-major:
            // 16 K rows of 128 bytes
            const uint64_t ad = kAMN ? sdesc_sw128_mn(a_addr + k * 2048, MN_BOX)
                                     : sdesc_sw128(a_addr + k * 32);
            const uint64_t bd = kBMN ? sdesc_sw128_mn(b_addr + k * 2048, MN_BOX)
                                     : sdesc_sw128(b_addr + k * 32);
            mma_bf16_ss(d_tmem, ad, bd, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
          }
          mma_commit(&empty[stage]);
          if (kb == kb1 - 1) mma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  } else if (warp >= 4) {
    pdl_wait();  // the epilogue reads the residual and writes outputs
    const int ew = warp - 4;  // TMEM lanes [32 ew, 32 ew + 32)
    uint8_t* boxes = out_boxes + ew * 2 * OUT_BOX;
    uint32_t buf = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      int mt, nt, kb0, kb1;
      decode_tile(tile, mt, nt, kb0, kb1);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = mt * BM + ew * 32 + lane_id();
      const bool row_ok = row < args.M;
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * kBN;
      if (ks_n > 1) {  // fp32 partial of this K split (rows < M only)
        float* P = args.ws + (static_cast<size_t>(tile % ks_n) * args.M + row) * args.N;
        for (int c = 0; c < kBN; c += 32) {
          uint32_t r[32];
          tmem_ld32(t_row + c, r);
          tmem_ld_wait();
          const int col = nt * kBN + c;
          if (row_ok && col < args.N) {
            if (col + 32 <= args.N && (args.N & 3) == 0) {
#pragma unroll
              for (int j = 0; j < 8; ++j)
                reinterpret_cast<float4*>(P + col)[j] =
                    make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (col + j < args.N) P[col + j] = __uint_as_float(r[j]);
            }
          }
        }
      } else if (kARows == BM && args.staged)
        epilogue_staged<kBN>(args, &tmC, t_row, mt * BM + ew * 32, nt, boxes, buf);
      else
        epilogue_row<kBN>(args, t_row, row, row_ok, nt, n_tiles);
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (kARows == BM && args.staged && lane_id() == 0) bulk_wait_all();
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<TMEM_COLS>(tmem_base);
}

// Split-K second pass: one thread per (row, output column); the splits are
// summed in order, then the epilogue is applied exactly as epilogue_row does
// (bias, GELU, SwiGLU over [gate128 | up128] tiles, residual, stores).
// Sum of the k_splits fp32 partials of (row, c) in split order, with every
// partial's load issued before the first add (the reductions are latency-bound).
constexpr int kMaxSplits = 16;
__device__ __forceinline__ float split_sum(const EpiArgs& args, int row, int c, size_t plane) {
  const float* p = args.ws + static_cast<size_t>(row) * args.N + c;
  float pv[kMaxSplits];
#pragma unroll
  for (int s = 0; s < kMaxSplits; ++s) pv[s] = s < args.k_splits ? p[s * plane] : 0.f;
  float v = pv[0];
#pragma unroll
  for (int s = 1; s < kMaxSplits; ++s)
    if (s < args.k_splits) v += pv[s];
  return v;
}

// Split-K reduction + bias + bf16 rounding (GEMM_EPI_BIAS_BF16), then RoPE on
// the q / k head blocks and the K | V copy into the generation row cache: one
// thread per (row, head block, frequency pair). The arithmetic is the plain
// reduction's followed by rope_kernel's (csrc/kernels_misc.cu), element for
// element, so the fused and unfused decode steps give identical bits.
__global__ void splitk_reduce_rope_append_kernel(EpiArgs args) {
  pdl_wait();
  pdl_trigger();
  const int nb = args.N / 128;
  const long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<long>(args.M) * nb * 64) return;
  const int row = static_cast<int>(i / (nb * 64)), rem = static_cast<int>(i % (nb * 64));
  const int hb = rem / 64, f = rem % 64;
  const int c0 = hb * 128 + f, c1 = c0 + 64;
  const size_t plane = static_cast<size_t>(args.M) * args.N;
  auto sum = [&](int c) { return split_sum(args, row, c, plane); };
  float v0 = sum(c0), v1 = sum(c1);
  if (args.bias) {
    v0 += args.bias[c0];
    v1 += args.bias[c1];
  }
  __nv_bfloat16 b0 = __float2bfloat16_rn(v0), b1 = __float2bfloat16_rn(v1);
  if (hb < args.n_rope_blocks) {
    float sn, cs;
    sincosf(__fmul_rn(static_cast<float>(args.pos[row]), args.inv_freq[f]), &sn, &cs);
    const float a = __bfloat162float(b0), b = __bfloat162float(b1);
    b0 = __float2bfloat16_rn(__fsub_rn(__fmul_rn(a, cs), __fmul_rn(b, sn)));
    b1 = __float2bfloat16_rn(__fadd_rn(__fmul_rn(b, cs), __fmul_rn(a, sn)));
  }
  __nv_bfloat16* crow = static_cast<__nv_bfloat16*>(args.C) + static_cast<size_t>(row) * args.ldc;
  crow[c0] = b0;
  crow[c1] = b1;
  if (c0 >= args.kv_col0 && c1 < args.kv_col0 + args.kvw) {
    __nv_bfloat16* kr =
        args.kv_rows + (static_cast<size_t>(*args.tdev) * args.M + row) * args.kvw - args.kv_col0;
    kr[c0] = b0;
    kr[c1] = b1;
  }
}

// Split-K reduction into the fp32 residual (GEMM_EPI_RESID_F32), then the
// RMSNorm of the updated row. One cluster of 4 CTAs per row, one column per
// thread (every split partial of the row in flight at once); the sum of
// squares is reduced per CTA in a fixed order and combined over the cluster
// through distributed shared memory in rank order, so every CTA derives the
// same scale and the result is deterministic.
__device__ __forceinline__ float ld_shared_cluster_f32(const float* p, uint32_t rank) {
  const uint32_t a = mapa_shared(smem_u32(p), rank);
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}
constexpr int kNormParts = 4;
__global__ void __cluster_dims__(kNormParts, 1, 1) __launch_bounds__(1024)
    splitk_reduce_resid_norm_kernel(EpiArgs args) {
  pdl_wait();
  pdl_trigger();
  __shared__ float s_warp[32];
  __shared__ float s_ss;
  const int part = blockIdx.x, row = blockIdx.y, tid = threadIdx.x;
  const int cols = args.N / kNormParts, col = part * cols + tid;
  const bool act = tid < cols;
  const size_t plane = static_cast<size_t>(args.M) * args.N;
  float h = 0.f;
  if (act) {
    float v = split_sum(args, row, col, plane);
    if (args.bias) v += args.bias[col];
    float* hp = args.resid + static_cast<size_t>(row) * args.ldr + col;
    h = *hp + v;
    *hp = h;
  }
  float ss = h * h;
#pragma unroll
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((tid & 31) == 0) s_warp[tid >> 5] = ss;
  __syncthreads();
  if (tid < 32) {
    float w = tid < static_cast<int>(blockDim.x >> 5) ? s_warp[tid] : 0.f;
#pragma unroll
    for (int o = 16; o; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
    if (tid == 0) s_ss = w;
  }
  cluster_sync();
  float tot = 0.f;
#pragma unroll
  for (int k = 0; k < kNormParts; ++k) tot += ld_shared_cluster_f32(&s_ss, k);
  const float r = rsqrtf(tot / static_cast<float>(args.N) + args.norm_eps);
  if (act)
    args.norm_out[static_cast<size_t>(row) * args.ld_norm + col] =
        __float2bfloat16_rn(args.norm_w[col] * (h * r));
  cluster_sync();  // peers may still read s_ss
}

__global__ void splitk_reduce_kernel(EpiArgs args) {
  pdl_wait();
  pdl_trigger();
  const bool swiglu = args.epi == GEMM_EPI_SWIGLU_BF16;
  const int n_out = swiglu ? args.N / 2 : args.N;
  const long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<long>(args.M) * n_out) return;
  const int row = static_cast<int>(i / n_out), col = static_cast<int>(i % n_out);
  const size_t plane = static_cast<size_t>(args.M) * args.N;
  auto sum = [&](int c) { return split_sum(args, row, c, plane); };
  if (swiglu) {
    const int c0 = (col / 128) * 256 + col % 128;
    const float g = sum(c0), u = sum(c0 + 128);
    static_cast<__nv_bfloat16*>(args.C)[static_cast<size_t>(row) * args.ldc + col] =
        __float2bfloat16_rn(silu(g) * u);
    return;
  }
  float v = sum(col);
  if (args.bias) v += args.bias[col];
  switch (args.epi) {
    case GEMM_EPI_RESID_F32:
      args.resid[static_cast<size_t>(row) * args.ldr + col] += v;
      break;
    case GEMM_EPI_STORE_F32:
      static_cast<float*>(args.C)[static_cast<size_t>(row) * args.ldc + col] = v;
      break;
    default:
      if (args.epi == GEMM_EPI_BIAS_GELU_BF16) v = gelu_tanh(v);
      static_cast<__nv_bfloat16*>(args.C)[static_cast<size_t>(row) * args.ldc + col] =
          __float2bfloat16_rn(v);
  }
}

// ---------------------------------------------------------------------------
// CTA-pair variant (cluster of 2, tcgen05 cta_group::2): a 256 x 256 tile per
// pair, M = 256 MMAs issued by the leader into both CTAs' TMEM. Each CTA TMA-
// loads its own 128 rows of A and its 128-row half of B (N), so per SM the
// smem operand reads drop from 96 B/clk (128x256 single-CTA tile: A 4 KB + B
// 8 KB per 128-clk MMA) to 64 B/clk and the TMA writes from 94 to 64 B/clk,
// under the 128 B/clk/SM smem port (tools/ubench/umma_rate.cu). Epilogue per
// CTA as in the single-CTA kernel (each CTA holds 128 rows x 256 columns).
// kRelay: each CTA's TMA completes on its own barrier and the follower's warp
// 3 forwards "stage landed" to the leader (instead of the 2-SM TMA form).
constexpr int P_STAGES = 6;
constexpr int P_HALF = BM * BK * 2;           // 16 KB: 128 rows x 64 K
constexpr int P_STAGE_BYTES = 2 * P_HALF;     // own A + own half of B
constexpr size_t P_SMEM_BYTES = 1024 + P_STAGES * P_STAGE_BYTES + OUT_BYTES + 512;

template <bool kRelay>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    gemm_bf16_pair(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC, EpiArgs args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* out_boxes = smem + P_STAGES * P_STAGE_BYTES;  // [4 warps][2][OUT_BOX]
  uint64_t* full = reinterpret_cast<uint64_t*>(out_boxes + OUT_BYTES);
  uint64_t* empty = full + P_STAGES;   // both CTAs: multicast MMA commit
  uint64_t* peer = empty + P_STAGES;   // leader: follower's stage landed (relay)
  uint64_t* tfull = peer + P_STAGES;   // [2] both CTAs: multicast MMA commit
  uint64_t* tempty = tfull + 2;        // [2] leader: 4 local + 4 remote epilogue warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = warp_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int m_tiles = (args.M + 2 * BM - 1) / (2 * BM);
  const int n_tiles = (args.N + BN - 1) / BN;
  const int num_tiles = m_tiles * n_tiles;
  const int k_blocks = (args.K + BK - 1) / BK;
  const int cl = static_cast<int>(blockIdx.x) >> 1, n_cl = static_cast<int>(gridDim.x) >> 1;

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (args.staged) tma_prefetch_desc(&tmC);
    for (int s = 0; s < P_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&peer[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_pair<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = cl; tile < num_tiles; tile += n_cl) {
        int mt, nt;
        tile_coords(tile, m_tiles, n_tiles, mt, nt);
        const int arow = mt * 2 * BM + static_cast<int>(rank) * BM;
        const int brow = nt * BN + static_cast<int>(rank) * BM;
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * P_STAGE_BYTES;
          if (kRelay) {
            mbar_arrive_expect_tx(&full[stage], P_STAGE_BYTES);
            tma_load_2d(sa, &tmA, &full[stage], kb * BK, arow);
            tma_load_2d(sa + P_HALF, &tmB, &full[stage], kb * BK, brow);
          } else {
            if (leader) mbar_arrive_expect_tx(&full[stage], 2 * P_STAGE_BYTES);
            tma_load_2d_2sm(sa, &tmA, &full[stage], kb * BK, arow);
            tma_load_2d_2sm(sa + P_HALF, &tmB, &full[stage], kb * BK, brow);
          }
          if (++stage == P_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1 && leader) {
    const uint32_t idesc = idesc_bf16_f32(2 * BM, BN);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = cl; tile < num_tiles; tile += n_cl) {
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = 0; kb < k_blocks; ++kb) {
        mbar_wait(&full[stage], phase);
        if (kRelay) mbar_wait(&peer[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a_addr = smem_u32(smem + stage * P_STAGE_BYTES);
          const uint32_t b_addr = a_addr + P_HALF;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            mma2_bf16_ss(d_tmem, sdesc_sw128(a_addr + k * 32), sdesc_sw128(b_addr + k * 32), idesc,
                         (kb | k) != 0);
          mma_commit_pair(&empty[stage], 3);
          if (kb == k_blocks - 1) mma_commit_pair(&tfull[acc], 3);
        }
        __syncwarp();
        if (++stage == P_STAGES) { stage = 0; phase ^= 1; }
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  } else if (kRelay && warp == 3 && !leader) {
    if (elect_one()) {  // forward this CTA's "stage landed" to the leader
      const uint32_t peer_l = mapa_shared(smem_u32(peer), 0);
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = cl; tile < num_tiles; tile += n_cl)
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&full[stage], phase);
          mbar_arrive_remote(peer_l + stage * 8);
          if (++stage == P_STAGES) { stage = 0; phase ^= 1; }
        }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    const uint32_t tempty_l = mapa_shared(smem_u32(tempty), 0);
    uint8_t* boxes = out_boxes + ew * 2 * OUT_BOX;
    uint32_t buf = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = cl; tile < num_tiles; tile += n_cl) {
      int mt, nt;
      tile_coords(tile, m_tiles, n_tiles, mt, nt);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int y = mt * 2 * BM + static_cast<int>(rank) * BM + ew * 32;
      const int row = y + lane_id();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * BN;
      if (args.staged)
        epilogue_staged(args, &tmC, t_row, y, nt, boxes, buf);
      else
        epilogue_row(args, t_row, row, row < args.M, nt, n_tiles);
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) {
        if (leader)
          mbar_arrive(&tempty[acc]);
        else
          mbar_arrive_remote(tempty_l + acc * 8);
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (args.staged && lane_id() == 0) bulk_wait_all();
  }

  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 2) tmem_dealloc_pair<TMEM_COLS>(tmem_base);
}

// Measured: in isolation the relayed CTA pair is the fastest on every LLM
// shape (tools/gemm_perf.py, interleaved: 16384x3584x3584 1219 vs 895
// TFLOP/s, SwiGLU 16384x37888x3584 1454 vs 1267), but inside the c4 step it
// draws the B200 deeper into its power cap: median SM clock 1500 -> 1400 MHz,
// GEMMs -80 ms, the attention that follows every GEMM +590 ms, step -4.5%
// (tools/ab_gemm.sh, same box). The single-CTA kernel is the default.
constexpr int kDefaultGemmImpl = 1;
constexpr int kSkinnyStages = 6, kSkinnyRows = 16;

}  // namespace

// Backward-pass GEMMs with MN-major operands (GemmArgs::a_mn / b_mn): the
// default single-CTA kernel, plain epilogues (bf16 / fp32 stores, fp32
// residual accumulate), staged TMA-store epilogue when aligned.
bool gemm_bf16_mn(const GemmArgs& g, cudaStream_t stream) {
  MRSP_REQUIRE(g.epi == GEMM_EPI_STORE_BF16 || g.epi == GEMM_EPI_STORE_F32 ||
                   g.epi == GEMM_EPI_RESID_F32 || g.epi == GEMM_EPI_BIAS_BF16,
               MRSP_INVALID_ARGUMENT, "gemm (MN-major operands): plain epilogues only");
  using K1 = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, EpiArgs);
  const int major = (g.a_mn ? 1 : 0) | (g.b_mn ? 2 : 0);
  const K1 kern = major == 1 ? gemm_bf16_tcgen05<STAGES, BM, 1>
                : major == 2 ? gemm_bf16_tcgen05<STAGES, BM, 2>
                             : gemm_bf16_tcgen05<STAGES, BM, 3>;
  static const bool attr_set = [] {
    for (K1 k : {gemm_bf16_tcgen05<STAGES, BM, 1>, gemm_bf16_tcgen05<STAGES, BM, 2>,
                 gemm_bf16_tcgen05<STAGES, BM, 3>})
      MRSP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(GemmCfg<STAGES, BM>::kSmem)));
    return true;
  }();
  (void)attr_set;
  CUtensorMap ta = g.a_mn ? make_tmap_bf16_2d(g.A, g.K, g.M, g.lda, BK, 64)
                          : make_tmap_bf16_2d(g.A, g.M, g.K, g.lda, BM, BK);
  CUtensorMap tb = g.b_mn ? make_tmap_bf16_2d(g.B, g.K, g.N, g.ldb, BK, 64)
                          : make_tmap_bf16_2d(g.B, g.N, g.K, g.ldb, BN, BK);
  const bool f32_out = g.epi == GEMM_EPI_STORE_F32 || g.epi == GEMM_EPI_RESID_F32;
  const uintptr_t out_addr = reinterpret_cast<uintptr_t>(g.epi == GEMM_EPI_RESID_F32 ? g.resid : g.C);
  const int ld_out = g.epi == GEMM_EPI_RESID_F32 ? g.ldr : g.ldc;
  const int vec_ok = (out_addr % 16 == 0) && (ld_out % (f32_out ? 4 : 8) == 0);
  EpiArgs e{};
  e.M = g.M;
  e.N = g.N;
  e.K = g.K;
  e.epi = g.epi;
  e.vec_ok = vec_ok;
  e.k_splits = 1;
  e.C = g.C;
  e.ldc = g.ldc;
  e.bias = g.bias;
  e.resid = g.resid;
  e.ldr = g.ldr;
  CUtensorMap tc = ta;
  if (vec_ok) {
    tc = g.epi == GEMM_EPI_RESID_F32 ? make_tmap_f32_2d(g.resid, g.M, g.N, g.ldr, 32, 32)
       : g.epi == GEMM_EPI_STORE_F32 ? make_tmap_f32_2d(g.C, g.M, g.N, g.ldc, 32, 32)
                                     : make_tmap_bf16_2d(g.C, g.M, g.N, g.ldc, 32, 64);
    e.staged = 1;
  }
  const int tiles = ((g.M + BM - 1) / BM) * ((g.N + BN - 1) / BN);
  kern<<<std::min(tiles, num_sms()), THREADS, GemmCfg<STAGES, BM>::kSmem, stream>>>(ta, tb, tc, e);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
  return false;
}

bool gemm_bf16(const GemmArgs& g, cudaStream_t stream) {
  MRSP_REQUIRE(g.M > 0 && g.N > 0 && g.K > 0, MRSP_INVALID_ARGUMENT, "gemm: empty problem");
  MRSP_REQUIRE((g.K % 8 == 0 || (g.a_mn && g.b_mn)) && g.lda % 8 == 0 && g.ldb % 8 == 0,
               MRSP_INVALID_ARGUMENT,
               "gemm: K and leading dims must be multiples of 8 (16-byte TMA pitch)");
  if (g.a_mn || g.b_mn) return gemm_bf16_mn(g, stream);
  if (g.epi == GEMM_EPI_SWIGLU_BF16)
    MRSP_REQUIRE(g.N % BN == 0, MRSP_INVALID_ARGUMENT, "gemm swiglu: N must be a multiple of 256");
  if (g.epi == GEMM_EPI_SWIGLU_BWD)
    MRSP_REQUIRE(g.N % BN == 0 && g.aux && g.aux_out && g.ld_aux % 8 == 0 &&
                     g.ld_aux_out % 8 == 0 && g.ldc % 8 == 0,
                 MRSP_INVALID_ARGUMENT, "gemm swiglu backward: bad arguments");
  if (g.epi == GEMM_EPI_RESID_F32)
    MRSP_REQUIRE(g.resid != nullptr, MRSP_INVALID_ARGUMENT, "gemm resid: null residual");
  static const bool attr_set = [] {  // thread-safe one-time setup (C-ABI callers may race)
    MRSP_CUDA(cudaFuncSetAttribute(gemm_bf16_tcgen05<STAGES, BM>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(GemmCfg<STAGES, BM>::kSmem)));
    MRSP_CUDA(cudaFuncSetAttribute(gemm_bf16_tcgen05<kSkinnyStages, kSkinnyRows>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(GemmCfg<kSkinnyStages, kSkinnyRows>::kSmem)));
    return true;
  }();
  (void)attr_set;
  // skinny ring for M <= 16 (MRSP_GEMM_SKINNY=0: off), plain epilogues only
  const char* env_skinny = std::getenv("MRSP_GEMM_SKINNY");
  const bool skinny_epi = g.epi == GEMM_EPI_STORE_BF16 || g.epi == GEMM_EPI_BIAS_BF16 ||
                          g.epi == GEMM_EPI_BIAS_GELU_BF16 || g.epi == GEMM_EPI_RESID_F32 ||
                          g.epi == GEMM_EPI_SWIGLU_BF16 || g.epi == GEMM_EPI_STORE_F32;
  const bool skinny = g.M <= kSkinnyRows && skinny_epi && !(env_skinny && std::atoi(env_skinny) == 0);
  CUtensorMap ta = make_tmap_bf16_2d(g.A, g.M, g.K, g.lda, skinny ? kSkinnyRows : BM, BK);
  CUtensorMap tb = make_tmap_bf16_2d(g.B, g.N, g.K, g.ldb, BN, BK);
  const bool f32_out = g.epi == GEMM_EPI_STORE_F32;
  const uintptr_t out_addr = reinterpret_cast<uintptr_t>(g.epi == GEMM_EPI_RESID_F32 ? g.resid : g.C);
  const int ld_out = g.epi == GEMM_EPI_RESID_F32 ? g.ldr : g.ldc;
  const int elem_per_16b = (f32_out || g.epi == GEMM_EPI_RESID_F32) ? 4 : 8;
  const int vec_ok = (out_addr % 16 == 0) && (ld_out % elem_per_16b == 0);
  EpiArgs e{g.M,     g.N,       g.K,     g.epi,     vec_ok,     0,          1, nullptr, g.C,
            g.ldc,
            g.bias,  g.resid,   g.ldr,   g.targets, g.part,     g.tgt_logit,
            g.pos,   g.inv_freq, g.n_rope_blocks, g.row0, g.route, g.peer_base, g.peer_ld,
            g.row_blocks, GEMM_POST_NONE, static_cast<__nv_bfloat16*>(g.kv_rows), g.kvw, g.kv_col0, g.tdev,
            g.norm_w, static_cast<__nv_bfloat16*>(g.norm_out), g.ld_norm, g.norm_eps,
            static_cast<const __nv_bfloat16*>(g.aux), g.ld_aux,
            static_cast<__nv_bfloat16*>(g.aux_out), g.ld_aux_out};
  if (g.post == GEMM_POST_ROPE_APPEND)
    MRSP_REQUIRE(g.epi == GEMM_EPI_BIAS_BF16 && g.N % 128 == 0 && g.pos && g.inv_freq &&
                     g.kv_rows && g.tdev && g.kvw % 128 == 0 && g.kv_col0 % 128 == 0,
                 MRSP_INVALID_ARGUMENT, "gemm rope/append: incomplete arguments");
  if (g.post == GEMM_POST_RMSNORM)
    MRSP_REQUIRE(g.epi == GEMM_EPI_RESID_F32 && g.norm_w && g.norm_out && g.N % 4 == 0 &&
                     g.ldr % 4 == 0,
                 MRSP_INVALID_ARGUMENT, "gemm resid/norm: incomplete arguments");
  if (g.epi == GEMM_EPI_QKV_SCATTER)
    MRSP_REQUIRE(g.N % 128 == 0 && g.bias && g.pos && g.inv_freq && g.route && g.peer_base &&
                     g.peer_ld,
                 MRSP_INVALID_ARGUMENT, "gemm qkv scatter: incomplete routing");
  if (g.epi == GEMM_EPI_LOGPROB_PARTIAL)
    MRSP_REQUIRE(g.targets && g.part && g.tgt_logit, MRSP_INVALID_ARGUMENT,
                 "gemm logprob: null targets/partials");
  // TMA-store epilogue for the plain / bias / GELU / SwiGLU / fp32 / residual
  // outputs when the output rows meet the tensor-map alignment rules
  // (MRSP_GEMM_EPI_DIRECT=1 keeps the per-row global-store epilogue).
  static const bool direct_env = [] {
    const char* v = std::getenv("MRSP_GEMM_EPI_DIRECT");
    return v != nullptr && std::atoi(v) != 0;
  }();
  CUtensorMap tc = ta;
  if (vec_ok && !direct_env) {
    switch (g.epi) {
      case GEMM_EPI_STORE_BF16:
      case GEMM_EPI_BIAS_BF16:
      case GEMM_EPI_BIAS_GELU_BF16:
        tc = make_tmap_bf16_2d(g.C, g.M, g.N, g.ldc, 32, 64);
        e.staged = 1;
        break;
      case GEMM_EPI_SWIGLU_BF16:
        tc = make_tmap_bf16_2d(g.C, g.M, g.N / 2, g.ldc, 32, 64);
        e.staged = 1;
        break;
      case GEMM_EPI_STORE_F32:
        tc = make_tmap_f32_2d(g.C, g.M, g.N, g.ldc, 32, 32);
        e.staged = 1;
        break;
      case GEMM_EPI_RESID_F32:
        tc = make_tmap_f32_2d(g.resid, g.M, g.N, g.ldr, 32, 32);
        e.staged = 1;
        break;
      default:
        break;
    }
  }
  // kernel choice (MRSP_GEMM_IMPL): 1 = single-CTA 128x256 tiles, 2 = CTA pair
  // with the 2-SM TMA form, 3 = CTA pair with relayed stage completion
  const char* env_impl = std::getenv("MRSP_GEMM_IMPL");
  const int impl = env_impl ? std::atoi(env_impl) : kDefaultGemmImpl;
  if (impl == 2 || impl == 3) {
    static const bool pair_attr = [] {
      MRSP_CUDA(cudaFuncSetAttribute(gemm_bf16_pair<false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(P_SMEM_BYTES)));
      MRSP_CUDA(cudaFuncSetAttribute(gemm_bf16_pair<true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(P_SMEM_BYTES)));
      return true;
    }();
    (void)pair_attr;
    CUtensorMap tbh = make_tmap_bf16_2d(g.B, g.N, g.K, g.ldb, BM, BK);  // 128-row halves of B
    const int tiles = ((g.M + 2 * BM - 1) / (2 * BM)) * ((g.N + BN - 1) / BN);
    const int grid = 2 * std::min(tiles, num_sms() / 2);
    if (impl == 3)
      gemm_bf16_pair<true><<<grid, THREADS, P_SMEM_BYTES, stream>>>(ta, tbh, tc, e);
    else
      gemm_bf16_pair<false><<<grid, THREADS, P_SMEM_BYTES, stream>>>(ta, tbh, tc, e);
    count_launch();
    MRSP_CUDA(cudaGetLastError());
    return false;
  }
  int tiles = ((g.M + BM - 1) / BM) * ((g.N + BN - 1) / BN);
  // split-K: one m tile, too few n tiles for the SMs, a workspace, a plain epilogue
  const int k_blocks = (g.K + BK - 1) / BK;
  const bool plain = g.epi == GEMM_EPI_STORE_BF16 || g.epi == GEMM_EPI_BIAS_BF16 ||
                     g.epi == GEMM_EPI_BIAS_GELU_BF16 || g.epi == GEMM_EPI_RESID_F32 ||
                     g.epi == GEMM_EPI_SWIGLU_BF16 || g.epi == GEMM_EPI_STORE_F32;
  if (g.splitk_ws && plain && g.M <= BM && 2 * tiles <= num_sms()) {
    const int splits = std::min({num_sms() / tiles, k_blocks / 4, 16});
    if (splits >= 2 && static_cast<size_t>(splits) * g.M * g.N * 4 <= g.splitk_ws_bytes) {
      e.k_splits = splits;
      e.ws = g.splitk_ws;
      e.staged = 0;
      tiles *= splits;
    }
  }
  // MRSP_GEMM_BN192=1: 192-wide tiles when N is a multiple of 192 but not of
  // 256 (SigLIP's 1152 / 3456: 6 / 18 full tiles instead of 4.5 / 13.5).
  // Measured neutral on the c4 tower (164.0-164.2 vs 164.4-164.9 ms), so off.
  static const bool bn192_env = [] {
    const char* v = std::getenv("MRSP_GEMM_BN192");
    return v && std::atoi(v) != 0;
  }();
  const bool bn192_epi = g.epi == GEMM_EPI_STORE_BF16 || g.epi == GEMM_EPI_BIAS_BF16 ||
                         g.epi == GEMM_EPI_BIAS_GELU_BF16 || g.epi == GEMM_EPI_RESID_F32 ||
                         g.epi == GEMM_EPI_STORE_F32;
  if (bn192_env && !skinny && e.k_splits <= 1 && bn192_epi && g.N % BN != 0 && g.N % 192 == 0) {
    static const bool attr192 = [] {
      MRSP_CUDA(cudaFuncSetAttribute(gemm_bf16_tcgen05<STAGES, BM, 0, 192>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(GemmCfg<STAGES, BM, 192>::kSmem)));
      return true;
    }();
    (void)attr192;
    CUtensorMap tb192 = make_tmap_bf16_2d(g.B, g.N, g.K, g.ldb, 192, BK);
    const int tiles192 = ((g.M + BM - 1) / BM) * (g.N / 192);
    launch_pdl(gemm_bf16_tcgen05<STAGES, BM, 0, 192>, dim3(std::min(tiles192, num_sms())),
               dim3(THREADS), GemmCfg<STAGES, BM, 192>::kSmem, stream, ta, tb192, tc, e);
    count_launch();
    MRSP_CUDA(cudaGetLastError());
    return false;
  }
  const int grid = std::min(tiles, num_sms());
  if (skinny) {
    e.staged = 0;
    launch_pdl(gemm_bf16_tcgen05<kSkinnyStages, kSkinnyRows>, dim3(grid), dim3(THREADS),
               GemmCfg<kSkinnyStages, kSkinnyRows>::kSmem, stream, ta, tb, tc, e);
  } else {
    launch_pdl(gemm_bf16_tcgen05<STAGES, BM>, dim3(grid), dim3(THREADS), GemmCfg<STAGES, BM>::kSmem,
               stream, ta, tb, tc, e);
  }
  count_launch();
  MRSP_CUDA(cudaGetLastError());
  if (e.k_splits <= 1) return false;
  if (g.post == GEMM_POST_ROPE_APPEND) {
    const long n = static_cast<long>(g.M) * (g.N / 128) * 64;
    launch_pdl(splitk_reduce_rope_append_kernel, dim3(static_cast<unsigned>((n + 255) / 256)),
               dim3(256), 0, stream, e);
  } else if (g.post == GEMM_POST_RMSNORM) {
    MRSP_REQUIRE(g.N % kNormParts == 0 && g.N / kNormParts <= 1024, MRSP_INVALID_ARGUMENT,
                 "gemm resid/norm: row too long");
    launch_pdl(splitk_reduce_resid_norm_kernel, dim3(kNormParts, g.M),
               dim3(((g.N / kNormParts + 31) / 32) * 32), 0, stream, e);
  } else {
    const long n = static_cast<long>(g.M) * (g.epi == GEMM_EPI_SWIGLU_BF16 ? g.N / 2 : g.N);
    launch_pdl(splitk_reduce_kernel, dim3(static_cast<unsigned>((n + 255) / 256)), dim3(256), 0,
               stream, e);
  }
  count_launch();
  MRSP_CUDA(cudaGetLastError());
  return g.post != GEMM_POST_NONE;
}

size_t gemm_splitk_ws_bytes(int M) {
  // splits x n tiles <= SMs, so splits x M x N <= SMs x M x BN
  return static_cast<size_t>(num_sms()) * M * BN * sizeof(float);
}

size_t lmhead_workspace_bytes(int M, int V) {
  const size_t n_tiles = (V + BN - 1) / BN;
  return (static_cast<size_t>(M) * n_tiles * sizeof(float2) + static_cast<size_t>(M) * 4 + 255) &
         ~size_t(255);
}

void lmhead_logprob(const void* X, int ldx, const void* W, int M, int V, int K,
                    const int32_t* targets, float* logprob, float* lse, void* ws, size_t ws_bytes,
                    cudaStream_t stream) {
  if (M <= 0) return;
  MRSP_REQUIRE(ws_bytes >= lmhead_workspace_bytes(M, V), MRSP_INVALID_ARGUMENT,
               "lmhead_logprob: workspace too small");
  const int n_tiles = (V + BN - 1) / BN;
  float2* part = static_cast<float2*>(ws);
  float* tgt = reinterpret_cast<float*>(part + static_cast<size_t>(M) * n_tiles);
  GemmArgs g{X, W, nullptr, M, V, K, ldx, K, 0, GEMM_EPI_LOGPROB_PARTIAL, nullptr, nullptr, 0};
  g.targets = targets;
  g.part = part;
  g.tgt_logit = tgt;
  gemm_bf16(g, stream);
  logprob_combine(part, n_tiles, tgt, M, logprob, lse, stream);
}

}  // namespace mrsp

extern "C" mrsp_status mrsp_op_gemm_bf16(const void* A, const void* B, void* C, int M, int N,
                                         int K, int lda, int ldb, int ldc, int epilogue,
                                         const float* bias, float* resid, int ldr, void* stream) {
  return mrsp::guard([&] {
    mrsp::require_device();
    mrsp::GemmArgs g{A, B, C, M, N, K, lda, ldb, ldc, epilogue, bias, resid, ldr};
    mrsp::gemm_bf16(g, static_cast<cudaStream_t>(stream));
  });
}

extern "C" mrsp_status mrsp_op_gemm_bf16_mn(const void* A, const void* B, void* C, int M, int N,
                                            int K, int lda, int ldb, int ldc, int a_mn, int b_mn,
                                            int epilogue, const float* bias, float* resid, int ldr,
                                            void* stream) {
  return mrsp::guard([&] {
    mrsp::require_device();
    mrsp::GemmArgs g{A, B, C, M, N, K, lda, ldb, ldc, epilogue, bias, resid, ldr};
    g.a_mn = a_mn;
    g.b_mn = b_mn;
    mrsp::gemm_bf16(g, static_cast<cudaStream_t>(stream));
  });
}

extern "C" mrsp_status mrsp_op_gemm_bf16_splitk(const void* A, const void* B, void* C, int M,
                                                int N, int K, int lda, int ldb, int ldc,
                                                int epilogue, const float* bias, float* resid,
                                                int ldr, void* workspace, size_t ws_bytes,
                                                void* stream) {
  return mrsp::guard([&] {
    mrsp::require_device();
    MRSP_REQUIRE(epilogue >= GEMM_EPI_STORE_BF16 && epilogue <= GEMM_EPI_STORE_F32,
                 MRSP_INVALID_ARGUMENT, "gemm splitk: plain epilogues only");
    mrsp::GemmArgs g{A, B, C, M, N, K, lda, ldb, ldc, epilogue, bias, resid, ldr};
    g.splitk_ws = static_cast<float*>(workspace);
    g.splitk_ws_bytes = workspace ? ws_bytes : 0;
    mrsp::gemm_bf16(g, static_cast<cudaStream_t>(stream));
  });
}

extern "C" size_t mrsp_gemm_splitk_workspace_bytes(int M) {
  return mrsp::gemm_splitk_ws_bytes(M);
}

extern "C" mrsp_status mrsp_op_lmhead_logprob(const void* X, int ldx, const void* W, int M, int V,
                                              int K, const int32_t* targets, float* logprob,
                                              float* lse, void* workspace, size_t ws_bytes,
                                              void* stream) {
  return mrsp::guard([&] {
    mrsp::require_device();
    mrsp::lmhead_logprob(X, ldx, W, M, V, K, targets, logprob, lse, workspace, ws_bytes,
                         static_cast<cudaStream_t>(stream));
  });
}

extern "C" size_t mrsp_lmhead_workspace_bytes(int M, int V) {
  return mrsp::lmhead_workspace_bytes(M, V);
}
