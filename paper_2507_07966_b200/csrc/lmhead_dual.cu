// lmhead_dual.cu — fused policy + reference LM head over the same scored tokens:
// one vocabulary sweep computes, per token, log pi_theta(y), log pi_ref(y) and the
// exact KL(pi_theta || pi_ref) over the whole vocabulary — the quantities the
// reference derives from two materialised [tokens x V] logit tensors in
// evaluate_from_logits (grpo.cpp:68-108: log_softmax, lp[y], exact KL at
// :94-96; per-position KL in policy.cpp:176-193). Logits never leave TMEM.
//
// Tile = 128 tokens x 256 vocab entries, BOTH models: two tcgen05 accumulators
// (2 x 256 TMEM columns). The TMA ring holds one model's k-block per stage
// (A 16 KB + B 32 KB) and alternates policy / reference, so 4 stages keep three
// 48 KB loads in flight behind the MMA (a 2-stage ring of 96 KB policy+reference
// stages kept one: 0.47 of the sustained peak). Epilogue: two warpgroups, each
// the tile's 128 rows (thread = token) over one 128-column half, online over
// its columns, with x = policy logit, y = reference logit,
//   m_x, s_x = sum e^(x - m_x), u = sum e^(x - m_x) (x - y), m_y, s_y = sum e^(y - m_y)
// plus the two target logits; a combine kernel merges the vocab tiles:
//   lse_x = M_x + log S_x,  KL = U / S_x - lse_x + lse_y,  lp = logit[y] - lse.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "common.h"
#include "backward.h"
#include "gemm.h"
#include "sm100.cuh"
#include "tma.h"

namespace mrsp {
namespace {

using namespace sm100;

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;  // one model's k-block
constexpr int THREADS = 384;                    // TMA, MMA, alloc, idle, 8 epilogue warps
constexpr int HALVES = 2;                       // epilogue column halves (one per warpgroup)
constexpr size_t SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + 256;

struct Part {  // per (token, vocab tile)
  float mx, sx, ux, my, sy;
};

struct DualArgs {
  int M, V, K, n_tiles;  // vocab tiles; partials per row = HALVES * n_tiles
  const int* targets;
  Part* part;
  float* tgt_x;
  float* tgt_y;
  // backward (kBwd): dJ/dlogits from the recomputed tiles (backward.h)
  const float* lse_x;
  const float* lse_y;
  const float* coef;
  const float* kl;
  float kw;
  __nv_bfloat16* G;
  int ldg;
};

// kBwd = false: the forward partials; true: the backward's dJ/dlogits tile
//   G = pi (kw (lp - lq - kl) - A) + A [v == y]   (grpo.cpp:152-180 per token)
template <bool kBwd>
__global__ void __launch_bounds__(THREADS, 1)
    lmhead_dual_tcgen05(const __grid_constant__ CUtensorMap tmAx, const __grid_constant__ CUtensorMap tmBx,
                        const __grid_constant__ CUtensorMap tmAy, const __grid_constant__ CUtensorMap tmBy,
                        DualArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
  const int warp = warp_id();
  const int m_tiles = (a.M + BM - 1) / BM;
  const int num_tiles = m_tiles * a.n_tiles;
  const int k_blocks = (a.K + BK - 1) / BK;

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmAx);
    tma_prefetch_desc(&tmBx);
    tma_prefetch_desc(&tmAy);
    tma_prefetch_desc(&tmBy);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 32 * 8);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int mt = tile % m_tiles, nt = tile / m_tiles;  // vocab-major: W tiles stream once
        for (int kb = 0; kb < k_blocks; ++kb) {
          for (int y = 0; y < 2; ++y) {  // policy k-block, then reference k-block
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* s = smem + stage * STAGE_BYTES;
            mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
            tma_load_2d(s, y ? &tmAy : &tmAx, &full[stage], kb * BK, mt * BM);
            tma_load_2d(s + A_BYTES, y ? &tmBy : &tmBx, &full[stage], kb * BK, nt * BN);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = idesc_bf16_f32(BM, BN);
    int stage = 0;
    uint32_t phase = 0;
    uint32_t tphase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      mbar_wait(tempty, tphase ^ 1);
      tc_fence_after();
      for (int kb = 0; kb < k_blocks; ++kb) {
        for (int y = 0; y < 2; ++y) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t s = smem_u32(smem + stage * STAGE_BYTES);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              mma_bf16_ss(tmem + y * BN, sdesc_sw128(s + k * 32), sdesc_sw128(s + A_BYTES + k * 32),
                          idesc, (kb | k) != 0);
            mma_commit(&empty[stage]);
            if (kb == k_blocks - 1 && y == 1) mma_commit(tfull);
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
      tphase ^= 1;
    }
  } else if (warp >= 4) {
    const int ew = (warp - 4) & 3, half = (warp - 4) >> 2;  // TMEM lane quarter, column half
    uint32_t tphase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int mt = tile % m_tiles, nt = tile / m_tiles;
      mbar_wait(tfull, tphase);
      tc_fence_after();
      const int row = mt * BM + ew * 32 + lane_id();
      const bool row_ok = row < a.M;
      const int tgt = row_ok ? a.targets[row] : -1;
      const uint32_t tr = tmem + (static_cast<uint32_t>(ew * 32) << 16);
      if constexpr (kBwd) {
        const float lx = row_ok ? a.lse_x[row] : 0.f, ly = row_ok ? a.lse_y[row] : 0.f;
        const float A = row_ok ? a.coef[row] : 0.f, klt = row_ok ? a.kl[row] : 0.f;
        for (int c = half * (BN / HALVES); c < (half + 1) * (BN / HALVES); c += 32) {
          uint32_t rx[32], ry[32];
          tmem_ld32(tr + c, rx);
          tmem_ld32(tr + BN + c, ry);
          tmem_ld_wait();
          const int col = nt * BN + c;
          if (row_ok && col < a.V) {
            uint32_t o[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              float gv[2];
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const float lp = __uint_as_float(rx[2 * j + e]) - lx;
                const float lq = __uint_as_float(ry[2 * j + e]) - ly;
                const float pi = __expf(lp);
                gv[e] = pi * (a.kw * (lp - lq - klt) - A) + (col + 2 * j + e == tgt ? A : 0.f);
              }
              o[j] = pack_bf16(gv[0], gv[1]);
            }
            __nv_bfloat16* dst = a.G + static_cast<size_t>(row) * a.ldg + col;
            if (col + 32 <= a.V) {
#pragma unroll
              for (int j = 0; j < 4; ++j)
                reinterpret_cast<uint4*>(dst)[j] = make_uint4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
            } else {
              const __nv_bfloat16* ob = reinterpret_cast<const __nv_bfloat16*>(o);
              for (int j = 0; col + j < a.V; ++j) dst[j] = ob[j];
            }
          }
        }
        tc_fence_before();
        mbar_arrive(tempty);
        tphase ^= 1;
        continue;
      }
      float mx = -INFINITY, sx = 0.f, ux = 0.f, my = -INFINITY, sy = 0.f;
      for (int c = half * (BN / HALVES); c < (half + 1) * (BN / HALVES); c += 32) {
        uint32_t rx[32], ry[32];
        tmem_ld32(tr + c, rx);
        tmem_ld32(tr + BN + c, ry);
        tmem_ld_wait();
        const int col = nt * BN + c;
        float cx = -INFINITY, cy = -INFINITY;
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (col + j < a.V) {
            cx = fmaxf(cx, __uint_as_float(rx[j]));
            cy = fmaxf(cy, __uint_as_float(ry[j]));
          }
        const float nx = fmaxf(mx, cx), ny = fmaxf(my, cy);
        const float fx = mx == -INFINITY ? 0.f : __expf(mx - nx);
        const float fy = my == -INFINITY ? 0.f : __expf(my - ny);
        float ax = sx * fx, au = ux * fx, ay = sy * fy;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float x = __uint_as_float(rx[j]), y = __uint_as_float(ry[j]);
          if (col + j < a.V) {
            const float ex = __expf(x - nx);
            ax += ex;
            au = fmaf(ex, x - y, au);
            ay += __expf(y - ny);
          }
          if (col + j == tgt) {
            a.tgt_x[row] = x;
            a.tgt_y[row] = y;
          }
        }
        mx = nx;
        my = ny;
        sx = ax;
        ux = au;
        sy = ay;
      }
      if (row_ok)
        a.part[(static_cast<size_t>(row) * a.n_tiles + nt) * HALVES + half] = Part{mx, sx, ux, my, sy};
      tc_fence_before();
      mbar_arrive(tempty);
      tphase ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

__global__ void lmhead_dual_combine(const Part* __restrict__ part, int n_tiles,
                                    const float* __restrict__ tgt_x, const float* __restrict__ tgt_y,
                                    int n, float* __restrict__ lp_x, float* __restrict__ lp_y,
                                    float* __restrict__ kl, float* __restrict__ lse_xo,
                                    float* __restrict__ lse_yo) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n) return;
  const Part* pr = part + static_cast<size_t>(warp) * n_tiles;
  float Mx = -INFINITY, My = -INFINITY;
  for (int t = lane; t < n_tiles; t += 32) {
    Mx = fmaxf(Mx, pr[t].mx);
    My = fmaxf(My, pr[t].my);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    Mx = fmaxf(Mx, __shfl_xor_sync(0xffffffffu, Mx, o));
    My = fmaxf(My, __shfl_xor_sync(0xffffffffu, My, o));
  }
  float Sx = 0.f, Ux = 0.f, Sy = 0.f;
  for (int t = lane; t < n_tiles; t += 32) {
    const float fx = expf(pr[t].mx - Mx);
    Sx += pr[t].sx * fx;
    Ux += pr[t].ux * fx;
    Sy += pr[t].sy * expf(pr[t].my - My);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    Sx += __shfl_xor_sync(0xffffffffu, Sx, o);
    Ux += __shfl_xor_sync(0xffffffffu, Ux, o);
    Sy += __shfl_xor_sync(0xffffffffu, Sy, o);
  }
  if (lane == 0) {
    const float lse_x = Mx + logf(Sx), lse_y = My + logf(Sy);
    lp_x[warp] = tgt_x[warp] - lse_x;
    lp_y[warp] = tgt_y[warp] - lse_y;
    kl[warp] = Ux / Sx - lse_x + lse_y;
    if (lse_xo) lse_xo[warp] = lse_x;
    if (lse_yo) lse_yo[warp] = lse_y;
  }
}

int sm_count() {
  static int n = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  return n;
}

}  // namespace

size_t lmhead_dual_workspace_bytes(int M, int V) {
  const size_t n_tiles = (V + BN - 1) / BN;
  return (static_cast<size_t>(M) * n_tiles * HALVES * sizeof(Part) + static_cast<size_t>(M) * 8 + 255) &
         ~size_t(255);
}

namespace {
void set_dual_attrs() {
  static const bool attr = [] {  // thread-safe one-time setup
    MRSP_CUDA(cudaFuncSetAttribute(lmhead_dual_tcgen05<false>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(SMEM_BYTES)));
    MRSP_CUDA(cudaFuncSetAttribute(lmhead_dual_tcgen05<true>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(SMEM_BYTES)));
    return true;
  }();
  (void)attr;
}
}  // namespace

void lmhead_dual_logprob_kl(const void* Xp, const void* Wp, const void* Xr, const void* Wr, int M,
                            int V, int K, const int32_t* targets, float* lp_p, float* lp_r,
                            float* kl, void* ws, size_t ws_bytes, cudaStream_t stream) {
  lmhead_dual_logprob_kl_lse(Xp, Wp, Xr, Wr, M, V, K, targets, lp_p, lp_r, kl, nullptr, nullptr,
                             ws, ws_bytes, stream);
}


void lmhead_dual_dlogits(const void* Xp, const void* Wp, const void* Xr, const void* Wr, int M,
                         int V, int K, const int32_t* targets, const float* coef, float kw,
                         const float* kl, const float* lse_p, const float* lse_r, void* G, int ldg,
                         cudaStream_t stream) {
  if (M <= 0) return;
  MRSP_REQUIRE(K % 8 == 0 && ldg % 8 == 0 && ldg >= V, MRSP_INVALID_ARGUMENT,
               "lmhead_dual_dlogits: K and ldg must be multiples of 8, ldg >= V");
  set_dual_attrs();
  DualArgs a{};
  a.M = M;
  a.V = V;
  a.K = K;
  a.n_tiles = (V + BN - 1) / BN;
  a.targets = targets;
  a.lse_x = lse_p;
  a.lse_y = lse_r;
  a.coef = coef;
  a.kl = kl;
  a.kw = kw;
  a.G = static_cast<__nv_bfloat16*>(G);
  a.ldg = ldg;
  CUtensorMap ax = make_tmap_bf16_2d(Xp, M, K, K, BM, BK);
  CUtensorMap bx = make_tmap_bf16_2d(Wp, V, K, K, BN, BK);
  CUtensorMap ay = make_tmap_bf16_2d(Xr, M, K, K, BM, BK);
  CUtensorMap by = make_tmap_bf16_2d(Wr, V, K, K, BN, BK);
  const int tiles = ((M + BM - 1) / BM) * a.n_tiles;
  lmhead_dual_tcgen05<true><<<std::min(tiles, sm_count()), THREADS, SMEM_BYTES, stream>>>(ax, bx, ay, by, a);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

void lmhead_dual_logprob_kl_lse(const void* Xp, const void* Wp, const void* Xr, const void* Wr,
                                int M, int V, int K, const int32_t* targets, float* lp_p,
                                float* lp_r, float* kl, float* lse_p, float* lse_r, void* ws,
                                size_t ws_bytes, cudaStream_t stream) {
  if (M <= 0) return;
  MRSP_REQUIRE(K % 8 == 0, MRSP_INVALID_ARGUMENT, "lmhead_dual: K must be a multiple of 8");
  MRSP_REQUIRE(ws_bytes >= lmhead_dual_workspace_bytes(M, V), MRSP_INVALID_ARGUMENT,
               "lmhead_dual: workspace too small");
  set_dual_attrs();
  DualArgs a{};
  a.M = M;
  a.V = V;
  a.K = K;
  a.n_tiles = (V + BN - 1) / BN;
  a.targets = targets;
  a.part = static_cast<Part*>(ws);
  a.tgt_x = reinterpret_cast<float*>(a.part + static_cast<size_t>(M) * a.n_tiles * HALVES);
  a.tgt_y = a.tgt_x + M;
  CUtensorMap ax = make_tmap_bf16_2d(Xp, M, K, K, BM, BK);
  CUtensorMap bx = make_tmap_bf16_2d(Wp, V, K, K, BN, BK);
  CUtensorMap ay = make_tmap_bf16_2d(Xr, M, K, K, BM, BK);
  CUtensorMap by = make_tmap_bf16_2d(Wr, V, K, K, BN, BK);
  const int tiles = ((M + BM - 1) / BM) * a.n_tiles;
  lmhead_dual_tcgen05<false><<<std::min(tiles, sm_count()), THREADS, SMEM_BYTES, stream>>>(ax, bx, ay, by, a);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
  lmhead_dual_combine<<<(M + 7) / 8, 256, 0, stream>>>(a.part, a.n_tiles * HALVES, a.tgt_x, a.tgt_y, M, lp_p,
                                                       lp_r, kl, lse_p, lse_r);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

}  // namespace mrsp

extern "C" size_t mrsp_lmhead_dual_workspace_bytes(int M, int V) {
  return mrsp::lmhead_dual_workspace_bytes(M, V);
}

extern "C" mrsp_status mrsp_op_lmhead_dual(const void* X_policy, const void* W_policy,
                                           const void* X_ref, const void* W_ref, int M, int V, int K,
                                           const int32_t* targets, float* logprob_policy,
                                           float* logprob_ref, float* kl, void* workspace,
                                           size_t ws_bytes, void* stream) {
  return mrsp::guard([&] {
    mrsp::require_device();
    mrsp::lmhead_dual_logprob_kl(X_policy, W_policy, X_ref, W_ref, M, V, K, targets, logprob_policy,
                                 logprob_ref, kl, workspace, ws_bytes,
                                 static_cast<cudaStream_t>(stream));
  });
}
