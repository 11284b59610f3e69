// gemm.cu — persistent, warp-specialised tcgen05 BF16 GEMM for sm_100a.
//
//   C[M,N] = epilogue( A[M,K] . B[N,K]^T )      A, B bf16 K-major, fp32 accumulate
//
// Roles (256 threads, one CTA per SM, grid = #SMs, static tile schedule):
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
// fp32 residual accumulate (hidden += A.B^T [+ bias]), plain bf16 / fp32 store.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "common.h"
#include "gemm.h"
#include "misc.h"
#include "sm100.cuh"
#include "tma.h"

namespace mrsp {
namespace {

using namespace sm100;

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int TMEM_COLS = 512;  // two 128x256 fp32 accumulators
constexpr int THREADS = 256;
constexpr size_t SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + 256;

struct EpiArgs {
  int M, N, K;
  int epi;
  int vec_ok;  // output/residual rows are 16-byte aligned -> vector stores
  void* C;
  int ldc;
  const float* bias;
  float* resid;
  int ldr;
  const int* targets;  // LOGPROB: target id per row
  float2* part;        // LOGPROB: [M][n_tiles] (tile max, sum exp(x - max))
  float* tgt_logit;    // LOGPROB: logit of the target per row
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

__device__ __forceinline__ float gelu_tanh(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  return 0.5f * x * (1.0f + tanhf(k0 * (x + k1 * x * x * x)));
}
__device__ __forceinline__ float silu(float x) { return x / (1.0f + __expf(-x)); }

__global__ void __launch_bounds__(THREADS, 1)
    gemm_bf16_tcgen05(const __grid_constant__ CUtensorMap tmA,
                      const __grid_constant__ CUtensorMap tmB, EpiArgs args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;   // [2]
  uint64_t* tempty = tfull + 2;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = warp_id();
  const int m_tiles = (args.M + BM - 1) / BM;
  const int n_tiles = (args.N + BN - 1) / BN;
  const int num_tiles = m_tiles * n_tiles;
  const int k_blocks = (args.K + BK - 1) / BK;

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
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

  if (warp == 0) {
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        int mt, nt;
        tile_coords(tile, m_tiles, n_tiles, mt, nt);
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
          tma_load_2d(sa, &tmA, &full[stage], kb * BK, mt * BM);
          tma_load_2d(sa + A_BYTES, &tmB, &full[stage], kb * BK, nt * BN);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = idesc_bf16_f32(BM, BN);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = 0; kb < k_blocks; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a_addr = smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t b_addr = a_addr + A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            mma_bf16_ss(d_tmem, sdesc_sw128(a_addr + k * 32), sdesc_sw128(b_addr + k * 32), idesc,
                        (kb | k) != 0);
          }
          mma_commit(&empty[stage]);
          if (kb == k_blocks - 1) mma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;  // TMEM lanes [32 ew, 32 ew + 32)
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      int mt, nt;
      tile_coords(tile, m_tiles, n_tiles, mt, nt);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = mt * BM + ew * 32 + lane_id();
      const bool row_ok = row < args.M;
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * BN;
      if (args.epi == GEMM_EPI_LOGPROB_PARTIAL) {
        // Fused vocabulary projection + log-softmax pieces: this 256-wide vocab
        // tile's (max, sum exp) per row and the target logit if it lies here.
        // Logits never leave TMEM/registers.
        const int tgt = row_ok ? args.targets[row] : -1;
        float m = -INFINITY, ssum = 0.f;
        for (int c = 0; c < BN; c += 32) {
          uint32_t r[32];
          tmem_ld32(t_row + c, r);
          tmem_ld_wait();
          const int col = nt * BN + c;
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
      } else if (args.epi == GEMM_EPI_SWIGLU_BF16) {
        // columns [0,128) are gate, [128,256) the matching up projections
        __nv_bfloat16* C = static_cast<__nv_bfloat16*>(args.C);
        for (int c = 0; c < BN / 2; c += 32) {
          uint32_t g[32], u[32];
          tmem_ld32(t_row + c, g);
          tmem_ld32(t_row + BN / 2 + c, u);
          tmem_ld_wait();
          const int col = nt * (BN / 2) + c;
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
        for (int c = 0; c < BN; c += 32) {
          uint32_t r[32];
          tmem_ld32(t_row + c, r);
          tmem_ld_wait();
          const int col = nt * BN + c;
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
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<TMEM_COLS>(tmem_base);
}

int num_sms() {
  static int n = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  return n;
}

}  // namespace

void gemm_bf16(const GemmArgs& g, cudaStream_t stream) {
  MRSP_REQUIRE(g.M > 0 && g.N > 0 && g.K > 0, MRSP_INVALID_ARGUMENT, "gemm: empty problem");
  MRSP_REQUIRE(g.K % 8 == 0 && g.lda % 8 == 0 && g.ldb % 8 == 0, MRSP_INVALID_ARGUMENT,
               "gemm: K and leading dims must be multiples of 8 (16-byte TMA pitch)");
  if (g.epi == GEMM_EPI_SWIGLU_BF16)
    MRSP_REQUIRE(g.N % BN == 0, MRSP_INVALID_ARGUMENT, "gemm swiglu: N must be a multiple of 256");
  if (g.epi == GEMM_EPI_RESID_F32)
    MRSP_REQUIRE(g.resid != nullptr, MRSP_INVALID_ARGUMENT, "gemm resid: null residual");
  static bool attr_set = false;
  if (!attr_set) {
    MRSP_CUDA(cudaFuncSetAttribute(gemm_bf16_tcgen05, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(SMEM_BYTES)));
    attr_set = true;
  }
  CUtensorMap ta = make_tmap_bf16_2d(g.A, g.M, g.K, g.lda, BM, BK);
  CUtensorMap tb = make_tmap_bf16_2d(g.B, g.N, g.K, g.ldb, BN, BK);
  const bool f32_out = g.epi == GEMM_EPI_STORE_F32;
  const uintptr_t out_addr = reinterpret_cast<uintptr_t>(g.epi == GEMM_EPI_RESID_F32 ? g.resid : g.C);
  const int ld_out = g.epi == GEMM_EPI_RESID_F32 ? g.ldr : g.ldc;
  const int elem_per_16b = (f32_out || g.epi == GEMM_EPI_RESID_F32) ? 4 : 8;
  const int vec_ok = (out_addr % 16 == 0) && (ld_out % elem_per_16b == 0);
  EpiArgs e{g.M,     g.N,       g.K,     g.epi,     vec_ok,     g.C,        g.ldc,
            g.bias,  g.resid,   g.ldr,   g.targets, g.part,     g.tgt_logit};
  if (g.epi == GEMM_EPI_LOGPROB_PARTIAL)
    MRSP_REQUIRE(g.targets && g.part && g.tgt_logit, MRSP_INVALID_ARGUMENT,
                 "gemm logprob: null targets/partials");
  const int tiles = ((g.M + BM - 1) / BM) * ((g.N + BN - 1) / BN);
  const int grid = std::min(tiles, num_sms());
  gemm_bf16_tcgen05<<<grid, THREADS, SMEM_BYTES, stream>>>(ta, tb, e);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
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
