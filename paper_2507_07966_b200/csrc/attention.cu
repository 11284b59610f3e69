// attention.cu — tcgen05 flash-attention forward for sm_100a (head dim 128).
//
// One CTA = one 128-query tile x one query head. K/V tiles of 128 keys stream
// through a 2-stage TMA ring; S = Q.K^T and O += P.V run on the tensor cores
// with fp32 accumulators in TMEM (S double-buffered, O resident for the
// whole KV sweep); the softmax warpgroup reads S with tcgen05.ld, keeps the
// running max / sum in registers, writes P (bf16) into swizzled smem for the
// P.V MMA and rescales O in TMEM only when the running max grows by > 2^8
// (lazy rescale; exact after the final 1/l normalisation).
//
// Roles (256 threads): warp 0 TMA, warp 1 MMA issuer, warp 2 TMEM allocator,
// warps 4-7 softmax / correction / epilogue (thread = query row).
//
// Masks (MR-SP packed sequence):
//   ATTN_CAUSAL_PREFIX: sequence = [prefix (Lp) | G rows of Lmax]; query q sees
//     key k iff k <= q and (k < Lp or row(k) == row(q)) — every rollout row
//     attends to the shared prompt prefix and causally to itself only.
//   ATTN_BLOCK_DIAG: bidirectional inside blocks of `blk` tokens (one video
//     frame of the vision tower), nothing across blocks.
// KV tiles with no visible (q,k) pair are skipped entirely; tiles that are
// fully visible skip the per-element mask.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "attention.h"
#include "common.h"
#include "sm100.cuh"
#include "tma.h"

namespace mrsp {
namespace {

using namespace sm100;

constexpr int TQ = 128, TK = 128, HD = 128;
constexpr int CHUNK = 128 * 64 * 2;       // one 128-row x 64-col bf16 SW128 block (16 KB)
constexpr int Q_BYTES = 2 * CHUNK;        // 32 KB
constexpr int KV_BYTES = 2 * CHUNK;       // 32 KB per K or V stage
constexpr int KV_STAGES = 2;
constexpr int P_BYTES = 2 * CHUNK;        // 32 KB
constexpr int OFF_Q = 0;
constexpr int OFF_K = OFF_Q + Q_BYTES;
constexpr int OFF_V = OFF_K + KV_STAGES * KV_BYTES;
constexpr int OFF_P = OFF_V + KV_STAGES * KV_BYTES;
constexpr int OFF_BAR = OFF_P + P_BYTES;
constexpr size_t SMEM_BYTES = 1024 + OFF_BAR + 256;
constexpr int THREADS = 256;
constexpr uint32_t TMEM_COLS = 512;  // S0 [0,128) S1 [128,256) O [256,384)
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 domain

struct MaskDev {
  int mode, L, Lp, Lmax, blk;
};

__device__ __forceinline__ int seg_of(int x, const MaskDev& m) { return (x - m.Lp) / m.Lmax; }

__device__ __forceinline__ bool visible(int q, int k, const MaskDev& m) {
  if (k >= m.L) return false;
  if (m.mode == ATTN_BLOCK_DIAG) return q / m.blk == k / m.blk;
  if (k > q) return false;
  return k < m.Lp || seg_of(k, m) == seg_of(q, m);
}

// 0 = skip, 1 = fully visible, 2 = needs the element mask.
__device__ __forceinline__ int tile_class(int q0, int kt, const MaskDev& m) {
  const int k0 = kt * TK, klast = k0 + TK - 1, qlast = q0 + TQ - 1;
  if (k0 >= m.L) return 0;
  if (m.mode == ATTN_BLOCK_DIAG) {
    const int kb0 = k0 / m.blk, kb1 = min(klast, m.L - 1) / m.blk;
    const int qb0 = q0 / m.blk, qb1 = qlast / m.blk;
    if (kb1 < qb0 || kb0 > qb1) return 0;
    return (kb0 == kb1 && qb0 == qb1 && kb0 == qb0 && klast < m.L) ? 1 : 2;
  }
  if (k0 > qlast) return 0;
  if (klast >= m.L) return 2;
  if (klast < m.Lp) return klast <= q0 ? 1 : 2;
  if (k0 < m.Lp) return 2;  // straddles the prefix / rows boundary
  if (qlast < m.Lp) return 0;
  const int sk0 = seg_of(k0, m), sk1 = seg_of(klast, m);
  const int qs0 = seg_of(max(q0, m.Lp), m), qs1 = seg_of(qlast, m);
  if (sk1 < qs0 || sk0 > qs1) return 0;
  return (sk0 == sk1 && qs0 == qs1 && sk0 == qs0 && q0 >= m.Lp && klast <= q0) ? 1 : 2;
}

__device__ __forceinline__ void kt_range(int q0, const MaskDev& m, int n_kt, int& lo, int& hi) {
  const int qlast = q0 + TQ - 1;
  if (m.mode == ATTN_BLOCK_DIAG) {
    lo = (q0 / m.blk) * m.blk / TK;
    hi = min(n_kt, ((qlast / m.blk + 1) * m.blk + TK - 1) / TK);
  } else {
    lo = 0;
    hi = min(n_kt, qlast / TK + 1);
  }
}

// Advances kt to the next non-skipped tile in [kt, hi); returns its class or 0.
__device__ __forceinline__ int next_tile(int q0, int& kt, int hi, const MaskDev& m) {
  for (; kt < hi; ++kt) {
    const int c = tile_class(q0, kt, m);
    if (c) return c;
  }
  return 0;
}

struct AttnArgs {
  int n_q_tiles, n_heads, q_per_kv;
  int q_col0, k_col0, v_col0, o_col0;
  __nv_bfloat16* O;
  int ldo;
  float scale_log2;
  MaskDev mask;
};

__global__ void __launch_bounds__(THREADS, 1)
    attn_fwd_tcgen05(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, AttnArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;   // [2]
  uint64_t* k_empty = bars + 3;  // [2]
  uint64_t* v_full = bars + 5;   // [2]
  uint64_t* v_empty = bars + 7;  // [2]
  uint64_t* s_full = bars + 9;   // [2]
  uint64_t* s_free = bars + 11;  // [2]
  uint64_t* p_full = bars + 13;
  uint64_t* pv_done = bars + 14;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);

  const int warp = warp_id();
  const int qt = a.n_q_tiles - 1 - static_cast<int>(blockIdx.x) / a.n_heads;  // heavy tiles first
  const int h = static_cast<int>(blockIdx.x) % a.n_heads;
  const int kvh = h / a.q_per_kv;
  const int q0 = qt * TQ;
  const int n_kt = (a.mask.L + TK - 1) / TK;
  int kt_lo, kt_hi;
  kt_range(q0, a.mask, n_kt, kt_lo, kt_hi);

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
      mbar_init(&s_full[s], 1);
      mbar_init(&s_free[s], 128);
    }
    mbar_init(p_full, 128);
    mbar_init(pv_done, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tO = tmem + 256;

  if (warp == 0) {
    if (elect_one()) {
      mbar_arrive_expect_tx(q_full, Q_BYTES);
      tma_load_2d(smem + OFF_Q, &tmQ, q_full, a.q_col0 + h * HD, q0);
      tma_load_2d(smem + OFF_Q + CHUNK, &tmQ, q_full, a.q_col0 + h * HD + 64, q0);
      int st = 0;
      uint32_t ph = 0;
      for (int kt = kt_lo; next_tile(q0, kt, kt_hi, a.mask); ++kt) {
        const int k0 = kt * TK;
        mbar_wait(&k_empty[st], ph ^ 1);
        mbar_arrive_expect_tx(&k_full[st], KV_BYTES);
        uint8_t* kd = smem + OFF_K + st * KV_BYTES;
        tma_load_2d(kd, &tmK, &k_full[st], a.k_col0 + kvh * HD, k0);
        tma_load_2d(kd + CHUNK, &tmK, &k_full[st], a.k_col0 + kvh * HD + 64, k0);
        mbar_wait(&v_empty[st], ph ^ 1);
        mbar_arrive_expect_tx(&v_full[st], KV_BYTES);
        uint8_t* vd = smem + OFF_V + st * KV_BYTES;
        tma_load_2d(vd, &tmV, &v_full[st], a.v_col0 + kvh * HD, k0);
        tma_load_2d(vd + CHUNK, &tmV, &v_full[st], a.v_col0 + kvh * HD + 64, k0);
        if (++st == KV_STAGES) { st = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc_s = idesc_bf16_f32(TQ, TK);
    const uint32_t idesc_o = idesc_bf16_f32_bmn(TQ, HD);
    const uint32_t q_addr = smem_u32(smem + OFF_Q);
    const uint32_t p_addr = smem_u32(smem + OFF_P);
    mbar_wait(q_full, 0);
    int it = 0;
    int st = 0;
    uint32_t ph = 0;
    int pst = 0;          // stage of the tile whose P.V is pending
    uint32_t pph = 0;
    bool pending = false;
    auto issue_pv = [&](int j) {
      mbar_wait(p_full, j & 1);
      mbar_wait(&v_full[pst], pph);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t v_addr = smem_u32(smem + OFF_V + pst * KV_BYTES);
#pragma unroll
        for (int kk = 0; kk < TK / 16; ++kk) {
          const uint64_t ad = sdesc_sw128(p_addr + (kk / 4) * CHUNK + (kk % 4) * 32);
          const uint64_t bd = sdesc_sw128_mn(v_addr + kk * 2048, CHUNK);
          mma_bf16_ss(tO, ad, bd, idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit(pv_done);
        mma_commit(&v_empty[pst]);
      }
      __syncwarp();
      if (++pst == KV_STAGES) { pst = 0; pph ^= 1; }
    };
    for (int kt = kt_lo; next_tile(q0, kt, kt_hi, a.mask); ++kt, ++it) {
      const int b = it & 1;
      mbar_wait(&k_full[st], ph);
      mbar_wait(&s_free[b], ((it >> 1) & 1) ^ 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t k_addr = smem_u32(smem + OFF_K + st * KV_BYTES);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk / 4) * CHUNK + (kk % 4) * 32;
          mma_bf16_ss(tmem + b * 128, sdesc_sw128(q_addr + off), sdesc_sw128(k_addr + off),
                      idesc_s, kk > 0 ? 1u : 0u);
        }
        mma_commit(&s_full[b]);
        mma_commit(&k_empty[st]);
      }
      __syncwarp();
      if (++st == KV_STAGES) { st = 0; ph ^= 1; }
      if (pending) issue_pv(it - 1);
      pending = true;
    }
    if (pending) issue_pv(it - 1);
  } else if (warp >= 4) {
    const int ew = warp - 4;
    const int r = ew * 32 + lane_id();  // query row in tile == TMEM lane
    const int q = q0 + r;
    const uint32_t lane_off = static_cast<uint32_t>(ew * 32) << 16;
    uint8_t* p_smem = smem + OFF_P;
    float m_run = -INFINITY, l_run = 0.f;
    int it = 0;
    for (int kt = kt_lo;; ++kt, ++it) {
      const int cls = next_tile(q0, kt, kt_hi, a.mask);
      if (!cls) break;
      const int b = it & 1;
      mbar_wait(&s_full[b], (it >> 1) & 1);
      tc_fence_after();
      float s[TK];
      {
        uint32_t r0[32], r1[32], r2[32], r3[32];
        const uint32_t base = tmem + lane_off + b * 128;
        tmem_ld32(base + 0, r0);
        tmem_ld32(base + 32, r1);
        tmem_ld32(base + 64, r2);
        tmem_ld32(base + 96, r3);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          s[j] = __uint_as_float(r0[j]);
          s[32 + j] = __uint_as_float(r1[j]);
          s[64 + j] = __uint_as_float(r2[j]);
          s[96 + j] = __uint_as_float(r3[j]);
        }
      }
      tc_fence_before();
      mbar_arrive(&s_free[b]);
      const int k0 = kt * TK;
      float mt = -INFINITY;
      if (cls == 2) {
#pragma unroll
        for (int j = 0; j < TK; ++j) {
          s[j] = visible(q, k0 + j, a.mask) ? s[j] * a.scale_log2 : -INFINITY;
          mt = fmaxf(mt, s[j]);
        }
      } else {
#pragma unroll
        for (int j = 0; j < TK; ++j) {
          s[j] *= a.scale_log2;
          mt = fmaxf(mt, s[j]);
        }
      }
      // P buffer and O are free once the previous P.V has completed.
      if (it > 0) mbar_wait(pv_done, (it - 1) & 1);
      tc_fence_after();
      // Lazy rescale: a row moves its reference max only when the tile max
      // exceeds it by 2^8. tcgen05.ld/st are warp-collective (.sync.aligned),
      // so the TMEM round trip runs for the whole warp when any lane needs it
      // (alpha = 1 for the others).
      const bool need = mt > m_run + RESCALE_THRESHOLD;
      if (__any_sync(0xffffffffu, need) && it > 0) {
        const float alpha = (need && m_run != -INFINITY) ? exp2f(m_run - mt) : 1.0f;
        if (need) l_run *= alpha;
#pragma unroll 1
        for (int c = 0; c < HD; c += 32) {
          uint32_t o[32];
          tmem_ld32(tO + lane_off + c, o);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * alpha);
          tmem_st32(tO + lane_off + c, o);
        }
        tmem_st_wait();
      }
      if (need) m_run = mt;
      const float m_use = m_run == -INFINITY ? 0.f : m_run;
      float lsum = 0.f;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          uint32_t w[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float p0 = exp2f(s[c * 64 + u * 8 + 2 * e] - m_use);
            const float p1 = exp2f(s[c * 64 + u * 8 + 2 * e + 1] - m_use);
            lsum += p0 + p1;
            w[e] = pack_bf16(p0, p1);
          }
          uint8_t* dst = p_smem + c * CHUNK + (r >> 3) * 1024 + (r & 7) * 128 + ((u ^ (r & 7)) << 4);
          *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
        }
      }
      l_run += lsum;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      mbar_arrive(p_full);
    }
    // epilogue: O / l -> bf16 global
    if (it > 0) mbar_wait(pv_done, (it - 1) & 1);
    tc_fence_after();
    const float inv_l = l_run > 0.f ? 1.0f / l_run : 0.f;
    const bool row_ok = q < a.mask.L;
    __nv_bfloat16* orow = a.O + static_cast<size_t>(q) * a.ldo + a.o_col0 + h * HD;
#pragma unroll 1
    for (int c = 0; c < HD; c += 32) {
      uint32_t o[32];
      tmem_ld32(tO + lane_off + c, o);
      tmem_ld_wait();
      if (row_ok) {
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j)
          pk[j] = pack_bf16(__uint_as_float(o[2 * j]) * inv_l, __uint_as_float(o[2 * j + 1]) * inv_l);
        uint4* dst = reinterpret_cast<uint4*>(orow + c);
#pragma unroll
        for (int j = 0; j < 4; ++j) dst[j] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<TMEM_COLS>(tmem);
}

}  // namespace

void attention_fwd(const AttnParams& p, cudaStream_t stream) {
  MRSP_REQUIRE(p.L > 0 && p.n_heads > 0 && p.q_per_kv > 0, MRSP_INVALID_ARGUMENT,
               "attention: empty problem");
  MRSP_REQUIRE(p.ldq % 8 == 0 && p.ldk % 8 == 0 && p.ldv % 8 == 0 && p.ldo % 8 == 0,
               MRSP_INVALID_ARGUMENT, "attention: leading dims must be multiples of 8");
  MRSP_REQUIRE(p.mode == ATTN_BLOCK_DIAG ? p.blk > 0 : (p.Lmax > 0 || p.Lp >= p.L),
               MRSP_INVALID_ARGUMENT, "attention: bad mask parameters");
  static bool attr = false;
  if (!attr) {
    MRSP_CUDA(cudaFuncSetAttribute(attn_fwd_tcgen05, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(SMEM_BYTES)));
    attr = true;
  }
  CUtensorMap tq = make_tmap_bf16_2d(p.Q, p.L, p.ldq, p.ldq, TQ, 64);
  CUtensorMap tk = make_tmap_bf16_2d(p.K, p.L, p.ldk, p.ldk, TK, 64);
  CUtensorMap tv = make_tmap_bf16_2d(p.V, p.L, p.ldv, p.ldv, TK, 64);
  AttnArgs a;
  a.n_q_tiles = (p.L + TQ - 1) / TQ;
  a.n_heads = p.n_heads;
  a.q_per_kv = p.q_per_kv;
  a.q_col0 = p.q_col0;
  a.k_col0 = p.k_col0;
  a.v_col0 = p.v_col0;
  a.o_col0 = p.o_col0;
  a.O = static_cast<__nv_bfloat16*>(p.O);
  a.ldo = p.ldo;
  a.scale_log2 = p.scale * 1.4426950408889634f;
  a.mask = MaskDev{p.mode, p.L, p.Lp, p.Lmax > 0 ? p.Lmax : 1, p.blk > 0 ? p.blk : 1};
  const int grid = a.n_q_tiles * a.n_heads;
  attn_fwd_tcgen05<<<grid, THREADS, SMEM_BYTES, stream>>>(tq, tk, tv, a);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

}  // namespace mrsp

extern "C" mrsp_status mrsp_op_attention(const void* Q, int ldq, int q_col0, const void* K, int ldk,
                                         int k_col0, const void* V, int ldv, int v_col0, void* O,
                                         int ldo, int o_col0, int L, int n_heads, int q_per_kv,
                                         float scale, int mode, int Lp, int Lmax, int blk,
                                         void* stream) {
  return mrsp::guard([&] {
    mrsp::require_device();
    mrsp::AttnParams p{Q, ldq, q_col0, K, ldk, k_col0, V, ldv, v_col0, O, ldo, o_col0,
                       L, n_heads, q_per_kv, scale, mode, Lp, Lmax, blk};
    mrsp::attention_fwd(p, static_cast<cudaStream_t>(stream));
  });
}
