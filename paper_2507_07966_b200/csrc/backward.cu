// backward.cu — the backward pass of the transformer-shaped MR-SP prefill
// ("backward through the SP prefill (GRPO/SFT gradients)";
// the reference differentiates its toy policy analytically, grpo.cpp:122-223
// through the GradAccumulator of policy.cpp:195-260 — here the same GRPO
// objective is differentiated through the Qwen-shaped decoder stack).
//
// Attention backward (head dim 128, the MR-SP causal-prefix mask), as two
// tcgen05 kernels so that every output is written once and the result is
// deterministic (no atomics; SP = k stays bit-identical to SP = 1):
//
//   attn_bwd_dq2   one CTA per (128-query tile, query head), sweeping the KV
//                  it sees in 64-key halves:  S = Q K^T, dP = dO V^T (TMEM,
//                  two buffers so the tensor core runs ahead of the softmax),
//                  then per element P = 2^(S scale log2e - lse), dS = P (dP - D)
//                  packed bf16 back into TMEM, and dQ += dS K (A operand from
//                  TMEM, K read MN-major from the same smem half). Q and dO,
//                  constant over the CTA, sit in TMEM as the S / dP A operands.
//   attn_bwd_dkdv4 one CTA per (128-key tile, kv head), sweeping the q_per_kv
//                  query heads x the 128-query tiles that see it:  S^T = K Q^T,
//                  dP^T = V dO^T, P^T and dS^T packed into TMEM, then
//                  dV += P^T dO and dK += dS^T Q (dO, Q read MN-major), the
//                  softmax handing P^T and dS^T over separately so that it
//                  runs behind dK(i-1), dP^T(i) and dV(i), S^T(i+1).
//                  (attn_bwd_dkdv2: 64-query halves over two S^T / dP^T
//                  buffers, MRSP_ATTN_BWD=2 / 3.)
//
// (attn_bwd_dq / attn_bwd_dkdv: the single-buffered 128-wide first version,
// MRSP_ATTN_BWD=1.) lse is the forward kernel's per-row log-sum-exp (scaled
// log2 domain, AttnParams::lse), D = rowsum(dO o O) (attn_bwd_prep). Roles as
// in the forward kernel: warp 0 TMA, warp 1 MMA issuer, warp 2 TMEM allocator,
// warps 4-11 two warpgroups that each take one half of the tile's columns.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "attn_common.cuh"
#include "backward.h"
#include "common.h"
#include "gemm.h"
#include "sm100.cuh"
#include "tma.h"

namespace mrsp {
namespace {

using namespace sm100;
using namespace attn_detail;

constexpr int CHUNK = 128 * 64 * 2;  // 128 rows x 64 bf16 columns, SW128 (16 KB)
constexpr int TILE = 2 * CHUNK;      // 128 x 128 bf16 (32 KB)
constexpr int THREADS = 384;

struct BwdArgs {
  int L, Lp, Lmax, n_heads, q_per_kv;
  int q_col0, k_col0, v_col0;  // columns of head 0 in qkv (and in dqkv)
  float scale, scale_log2;
  const float* lse;  // [n_heads][ld_stat]
  const float* D;
  int ld_stat;
  __nv_bfloat16* dqkv;
  int ld_dqkv;
  // query-row split (common.h attn_row_part): only the 256-row query blocks of
  // part row_part of row_parts (dQ rows; the dK / dV are then partial sums)
  int row_parts, row_part, n_blocks, n_local_blocks;
  // optional fp32 dK | dV output [L][ld_dkv32] (dk of local kv head g at
  // 128 g, dv at (n_kv + g) 128) instead of bf16 into dqkv: the partials of a
  // kv head shared by several ranks, summed before their single rounding
  float* dkv32;
  int ld_dkv32;
  // raw rows (the dQ kernel reads its constant A operands Q / dO into TMEM)
  const __nv_bfloat16* qkv;
  int ld_qkv;
  const __nv_bfloat16* dO;
  int ld_do;
};

// Query tile of dQ-kernel CTA index `rem` (kv-head-major order handled by the
// caller): heaviest tiles first; with a row split, the part's blocks in
// attn_row_block order.
__device__ __forceinline__ int dq_tile(int lt, const BwdArgs& a, int n_qt) {
  if (a.row_parts <= 1) return n_qt - 1 - lt;
  return attn_row_block(lt >> 1, a.row_part, a.n_blocks, a.row_parts) * 2 + (lt & 1);
}
__device__ __forceinline__ bool own_rows(int q, const BwdArgs& a) {
  return a.row_parts <= 1 || attn_row_part(q / ATTN_ROW_BLOCK, a.n_blocks, a.row_parts) == a.row_part;
}

__device__ __forceinline__ MaskDev mask_of(const BwdArgs& a) {
  return MaskDev{ATTN_CAUSAL_PREFIX, a.L, a.Lp, a.Lmax, 1};
}

// Per-phase timeline of one dK / dV CTA (dev tool tools/ubench/bwd_trace.cu
// builds this file with MRSP_BWD_TRACE): clock() stamps of lane 0 per warp.
#ifdef MRSP_BWD_TRACE
constexpr int kBTraceCap = 4096;
__device__ uint64_t g_bwd_trace[12][kBTraceCap];
__device__ int g_bwd_trace_n[12];
__device__ int g_bwd_trace_cta;
__device__ int g_bwd_trace_kernel;  // 0: dK / dV, 1: dQ
#define BTRACE_INIT(kid) \
  const bool btrace_on = blockIdx.x == g_bwd_trace_cta && g_bwd_trace_kernel == (kid); \
  int btrace_n = 0
#define BTRACE(ev, it)                                                                            \
  do {                                                                                            \
    if (btrace_on && (threadIdx.x & 31) == 0 && btrace_n < kBTraceCap)                            \
      g_bwd_trace[threadIdx.x >> 5][btrace_n++] = (static_cast<uint64_t>(ev) << 56) |              \
                                                  (static_cast<uint64_t>((it) & 0xffffff) << 32) | \
                                                  static_cast<uint32_t>(clock());                 \
  } while (0)
#define BTRACE_FINISH \
  if (btrace_on && (threadIdx.x & 31) == 0) g_bwd_trace_n[threadIdx.x >> 5] = btrace_n
#else
#define BTRACE_INIT(kid)
#define BTRACE(ev, it) \
  do {                 \
  } while (0)
#define BTRACE_FINISH
#endif

// K-major SW128 operand: 16-element K step kk of a 128 x 128 tile (two 64-col chunks)
__device__ __forceinline__ uint32_t kmajor_off(int kk) { return (kk / 4) * CHUNK + (kk % 4) * 32; }

// ----------------------------------------------------------------------------
// dQ: one CTA per (query tile, query head). Work order: kv-head-major, then the
// query tiles heaviest (longest key sweep) first, then the heads of the group.
constexpr int DQ_RING = 4;  // K / V single-tile slots
constexpr int DQ_OFF_Q = 0, DQ_OFF_DO = TILE, DQ_OFF_RING = 2 * TILE;
constexpr int DQ_OFF_BAR = DQ_OFF_RING + DQ_RING * TILE;
constexpr size_t DQ_SMEM = 1024 + DQ_OFF_BAR + 256;

__global__ void __launch_bounds__(THREADS, 1)
    attn_bwd_dq(const __grid_constant__ CUtensorMap tmQKV, const __grid_constant__ CUtensorMap tmDO,
                BwdArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + DQ_OFF_BAR);
  uint64_t* q_full = bars;
  uint64_t* r_full = bars + 1;              // [DQ_RING]
  uint64_t* r_empty = bars + 1 + DQ_RING;   // [DQ_RING]
  uint64_t* s_full = bars + 1 + 2 * DQ_RING;
  uint64_t* ds_full = s_full + 1;
  uint64_t* dq_done = s_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 3);

  const int warp = warp_id();
  const MaskDev m = mask_of(a);
  const int n_qt = (a.L + TQ - 1) / TQ, n_kt = (a.L + TK - 1) / TK;
  const int n_tiles = a.row_parts > 1 ? 2 * a.n_local_blocks : n_qt;
  const int per_kv = n_tiles * a.q_per_kv;
  const int kvh = blockIdx.x / per_kv;
  const int rem = blockIdx.x - kvh * per_kv;
  const int qt = dq_tile(rem / a.q_per_kv, a, n_qt);
  const int h = kvh * a.q_per_kv + rem % a.q_per_kv;
  const int q0 = qt * TQ;
  const int kt_hi = min(n_kt, (q0 + TQ - 1) / TK + 1);
  auto next = [&](int& kt) {  // next visible KV tile at or after kt (class, 0 = done)
    for (; kt < kt_hi; ++kt) {
      const int c = tile_class(q0, kt, m);
      if (c) return c;
    }
    return 0;
  };

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmQKV);
    tma_prefetch_desc(&tmDO);
    mbar_init(q_full, 1);
    for (int s = 0; s < DQ_RING; ++s) {
      mbar_init(&r_full[s], 1);
      mbar_init(&r_empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(ds_full, 256);
    mbar_init(dq_done, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;  // S [0,128) dP [128,256) dQ [256,384)

  if (warp < 4) {
    reg_dealloc<56>();
    if (warp == 0) {
      if (elect_one()) {
        mbar_arrive_expect_tx(q_full, 2 * TILE);
        for (int c = 0; c < 2; ++c) {
          tma_load_2d(smem + DQ_OFF_Q + c * CHUNK, &tmQKV, q_full, a.q_col0 + h * HD + c * 64, q0);
          tma_load_2d(smem + DQ_OFF_DO + c * CHUNK, &tmDO, q_full, h * HD + c * 64, q0);
        }
        int slot = 0;
        uint32_t ph = 0;
        for (int kt = 0; next(kt); ++kt) {
          for (int kv = 0; kv < 2; ++kv) {  // K_j then V_j
            mbar_wait(&r_empty[slot], ph ^ 1);
            mbar_arrive_expect_tx(&r_full[slot], TILE);
            const int col = (kv ? a.v_col0 : a.k_col0) + kvh * HD;
            uint8_t* dst = smem + DQ_OFF_RING + slot * TILE;
            tma_load_2d(dst, &tmQKV, &r_full[slot], col, kt * TK);
            tma_load_2d(dst + CHUNK, &tmQKV, &r_full[slot], col + 64, kt * TK);
            if (++slot == DQ_RING) { slot = 0; ph ^= 1; }
          }
        }
      }
    } else if (warp == 1) {
      const uint32_t idesc_s = idesc_bf16_f32(TQ, TK);
      const uint32_t idesc_o = idesc_bf16_f32_bmn(TQ, HD);
      const uint32_t q_addr = smem_u32(smem + DQ_OFF_Q), do_addr = smem_u32(smem + DQ_OFF_DO);
      const uint32_t ring = smem_u32(smem + DQ_OFF_RING);
      mbar_wait(q_full, 0);
      int slot = 0, it = 0;
      uint32_t ph = 0;
      for (int kt = 0; next(kt); ++kt, ++it) {
        const int ks = slot;
        mbar_wait(&r_full[ks], ph);
        if (++slot == DQ_RING) { slot = 0; ph ^= 1; }
        const int vs = slot;
        mbar_wait(&r_full[vs], ph);
        if (++slot == DQ_RING) { slot = 0; ph ^= 1; }
        const uint32_t k_addr = ring + ks * TILE, v_addr = ring + vs * TILE;
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk)
            mma_bf16_ss(tmem, sdesc_sw128(q_addr + kmajor_off(kk)),
                        sdesc_sw128(k_addr + kmajor_off(kk)), idesc_s, kk > 0 ? 1u : 0u);
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk)
            mma_bf16_ss(tmem + 128, sdesc_sw128(do_addr + kmajor_off(kk)),
                        sdesc_sw128(v_addr + kmajor_off(kk)), idesc_s, kk > 0 ? 1u : 0u);
          mma_commit(s_full);
          mma_commit(&r_empty[vs]);
        }
        __syncwarp();
        mbar_wait(ds_full, it & 1);
        tc_fence_after();
        if (elect_one()) {
          // dQ += dS . K: dS packed bf16 in S columns [0,32) (keys 0-63) and
          // [64,96) (keys 64-127); K_j read MN-major (hd contiguous)
#pragma unroll
          for (int kk = 0; kk < TK / 16; ++kk)
            mma_bf16_ts(tmem + 256, tmem + (kk / 4) * 64 + (kk % 4) * 8,
                        sdesc_sw128_mn(k_addr + kk * 2048, CHUNK), idesc_o,
                        (it > 0 || kk > 0) ? 1u : 0u);
          mma_commit(&r_empty[ks]);
        }
        __syncwarp();
      }
      if (elect_one()) mma_commit(dq_done);
      __syncwarp();
    }
  } else {
    reg_alloc<200>();
    const int hf = (warp - 4) >> 2;     // key half of the tile this warpgroup handles
    const int ew = (warp - 4) & 3;      // TMEM lane quarter
    const int r = ew * 32 + lane_id();  // query row in the tile
    const int q = q0 + r;
    const bool row_ok = q < a.L;
    const uint32_t lane_off = static_cast<uint32_t>(ew * 32) << 16;
    const float lse = row_ok ? a.lse[static_cast<size_t>(h) * a.ld_stat + q] : INFINITY;
    const float Dq = row_ok ? a.D[static_cast<size_t>(h) * a.ld_stat + q] : 0.f;
    const float sl2 = a.scale_log2;
    const int k_end = min(q + 1, a.L), k_mid = a.Lp;
    const int k_lo = q >= a.Lp ? a.Lp + seg_of(q, m) * a.Lmax : 0;
    int it = 0;
    for (int kt = 0;; ++kt, ++it) {
      const int cls = next(kt);
      if (!cls) break;
      mbar_wait(s_full, it & 1);
      tc_fence_after();
      uint32_t s0[32], s1[32], d0[32], d1[32];
      tmem_ld32(tmem + lane_off + hf * 64, s0);
      tmem_ld32(tmem + lane_off + hf * 64 + 32, s1);
      tmem_ld32(tmem + lane_off + 128 + hf * 64, d0);
      tmem_ld32(tmem + lane_off + 128 + hf * 64 + 32, d1);
      tmem_ld_wait();
      const int kb = kt * TK + hf * 64;
      uint32_t vis0 = 0xffffffffu, vis1 = 0xffffffffu;
      if (cls == 2) {
        vis0 = lt_bits(k_end, kb) & (lt_bits(k_mid, kb) | ~lt_bits(k_lo, kb));
        vis1 = lt_bits(k_end, kb + 32) & (lt_bits(k_mid, kb + 32) | ~lt_bits(k_lo, kb + 32));
      }
      uint32_t w[32];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        float p[4], g[4];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int j = 2 * i + e;
          p[e] = ((vis0 >> j) & 1u) ? exp2_mufu(__uint_as_float(s0[j]) * sl2 - lse) : 0.f;
          p[2 + e] = ((vis1 >> j) & 1u) ? exp2_mufu(__uint_as_float(s1[j]) * sl2 - lse) : 0.f;
          g[e] = p[e] * (__uint_as_float(d0[j]) - Dq);
          g[2 + e] = p[2 + e] * (__uint_as_float(d1[j]) - Dq);
        }
        w[i] = pack_bf16(g[0], g[1]);
        w[16 + i] = pack_bf16(g[2], g[3]);
      }
      tmem_st32(tmem + lane_off + hf * 64, w);
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(ds_full);
    }
    // epilogue: dQ (scaled) -> bf16, this warpgroup's 64 head columns
    __nv_bfloat16* out = a.dqkv + static_cast<size_t>(q) * a.ld_dqkv + a.q_col0 + h * HD + hf * 64;
    if (it > 0) {
      mbar_wait(dq_done, 0);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < 64; c += 32) {
        uint32_t o[32];
        tmem_ld32(tmem + lane_off + 256 + hf * 64 + c, o);
        tmem_ld_wait();
        if (row_ok) {
          uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 16; ++j)
            pk[j] = pack_bf16(__uint_as_float(o[2 * j]) * a.scale, __uint_as_float(o[2 * j + 1]) * a.scale);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            reinterpret_cast<uint4*>(out + c)[j] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
        }
      }
    } else if (row_ok) {
      for (int c = 0; c < 64; c += 8) *reinterpret_cast<uint4*>(out + c) = make_uint4(0, 0, 0, 0);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// ----------------------------------------------------------------------------
// dK, dV: one CTA per (key tile, kv head), key tiles in ascending order (the
// prefix keys, seen by every later query, are the heaviest).
constexpr int KV_RING = 2;                       // (Q_i, dO_i, lse_i, D_i) stages
constexpr int KV_STAT = 2 * 128 * 4;             // lse + D of one query tile
constexpr int KV_STAGE = 2 * TILE + KV_STAT;     // 64 KB + 1 KB
constexpr int KV_OFF_K = 0, KV_OFF_V = TILE, KV_OFF_RING = 2 * TILE;
constexpr int KV_OFF_BAR = KV_OFF_RING + KV_RING * KV_STAGE;
constexpr size_t KV_SMEM = 1024 + KV_OFF_BAR + 256;
static_assert(KV_STAGE % 1024 == 0, "stages stay 1024-byte aligned (SW128 atoms)");

__global__ void __launch_bounds__(THREADS, 1)
    attn_bwd_dkdv(const __grid_constant__ CUtensorMap tmQKV, const __grid_constant__ CUtensorMap tmDO,
                  const __grid_constant__ CUtensorMap tmLSE, const __grid_constant__ CUtensorMap tmD,
                  BwdArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + KV_OFF_BAR);
  uint64_t* kv_full = bars;
  uint64_t* r_full = bars + 1;             // [KV_RING]
  uint64_t* r_empty = bars + 1 + KV_RING;  // [KV_RING]
  uint64_t* s_full = bars + 1 + 2 * KV_RING;
  uint64_t* ds_full = s_full + 1;
  uint64_t* acc_done = s_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 3);

  const int warp = warp_id();
  const MaskDev m = mask_of(a);
  const int n_qt = (a.L + TQ - 1) / TQ, n_kt = (a.L + TK - 1) / TK;
  const int kvh = blockIdx.x / n_kt;
  const int kt = blockIdx.x - kvh * n_kt;
  const int k0 = kt * TK;
  // query tiles that can see this key tile: from the diagonal up to the end of
  // the sequence (the tile holds a prefix key) or of the last key's rollout row
  const int klast = min(k0 + TK - 1, a.L - 1);
  const int q_end = k0 < a.Lp ? a.L : min(a.L, a.Lp + (seg_of(klast, m) + 1) * a.Lmax);
  const int qt_lo = k0 / TQ, qt_hi = min(n_qt, (q_end + TQ - 1) / TQ);
  const int n_items = (qt_hi - qt_lo) * a.q_per_kv;  // (head, query tile), head-minor
  auto next = [&](int& i, int& hh, int& qt) {  // next visible item at or after i
    for (; i < n_items; ++i) {
      qt = qt_lo + i / a.q_per_kv;
      hh = i % a.q_per_kv;
      const int c = tile_class(qt * TQ, kt, m);
      if (c) return c;
    }
    return 0;
  };

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmQKV);
    tma_prefetch_desc(&tmDO);
    tma_prefetch_desc(&tmLSE);
    tma_prefetch_desc(&tmD);
    mbar_init(kv_full, 1);
    for (int s = 0; s < KV_RING; ++s) {
      mbar_init(&r_full[s], 1);
      mbar_init(&r_empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(ds_full, 256);
    mbar_init(acc_done, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;  // S^T [0,128) dP^T [128,256) dV [256,384) dK [384,512)

  if (warp < 4) {
    reg_dealloc<56>();
    if (warp == 0) {
      if (elect_one()) {
        mbar_arrive_expect_tx(kv_full, 2 * TILE);
        for (int c = 0; c < 2; ++c) {
          tma_load_2d(smem + KV_OFF_K + c * CHUNK, &tmQKV, kv_full, a.k_col0 + kvh * HD + c * 64, k0);
          tma_load_2d(smem + KV_OFF_V + c * CHUNK, &tmQKV, kv_full, a.v_col0 + kvh * HD + c * 64, k0);
        }
        int slot = 0;
        uint32_t ph = 0;
        int hh, qt;
        for (int i = 0; next(i, hh, qt); ++i) {
          const int h = kvh * a.q_per_kv + hh;
          mbar_wait(&r_empty[slot], ph ^ 1);
          mbar_arrive_expect_tx(&r_full[slot], KV_STAGE);
          uint8_t* st = smem + KV_OFF_RING + slot * KV_STAGE;
          for (int c = 0; c < 2; ++c) {
            tma_load_2d(st + c * CHUNK, &tmQKV, &r_full[slot], a.q_col0 + h * HD + c * 64, qt * TQ);
            tma_load_2d(st + TILE + c * CHUNK, &tmDO, &r_full[slot], h * HD + c * 64, qt * TQ);
          }
          tma_load_2d(st + 2 * TILE, &tmLSE, &r_full[slot], qt * TQ, h);
          tma_load_2d(st + 2 * TILE + 512, &tmD, &r_full[slot], qt * TQ, h);
          if (++slot == KV_RING) { slot = 0; ph ^= 1; }
        }
      }
    } else if (warp == 1) {
      const uint32_t idesc_s = idesc_bf16_f32(TK, TQ);
      const uint32_t idesc_o = idesc_bf16_f32_bmn(TK, HD);
      const uint32_t k_addr = smem_u32(smem + KV_OFF_K), v_addr = smem_u32(smem + KV_OFF_V);
      const uint32_t ring = smem_u32(smem + KV_OFF_RING);
      mbar_wait(kv_full, 0);
      int slot = 0, it = 0;
      uint32_t ph = 0;
      int hh, qt;
      for (int i = 0; next(i, hh, qt); ++i, ++it) {
        mbar_wait(&r_full[slot], ph);
        tc_fence_after();
        const uint32_t q_addr = ring + slot * KV_STAGE, do_addr = q_addr + TILE;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk)
            mma_bf16_ss(tmem, sdesc_sw128(k_addr + kmajor_off(kk)),
                        sdesc_sw128(q_addr + kmajor_off(kk)), idesc_s, kk > 0 ? 1u : 0u);
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk)
            mma_bf16_ss(tmem + 128, sdesc_sw128(v_addr + kmajor_off(kk)),
                        sdesc_sw128(do_addr + kmajor_off(kk)), idesc_s, kk > 0 ? 1u : 0u);
          mma_commit(s_full);
        }
        __syncwarp();
        mbar_wait(ds_full, it & 1);
        tc_fence_after();
        if (elect_one()) {
          // dV += P^T . dO, dK += dS^T . Q (A from TMEM, packed pairs in
          // columns [0,32) + [64,96) of S^T / dP^T; B read MN-major)
#pragma unroll
          for (int kk = 0; kk < TQ / 16; ++kk) {
            const uint32_t acol = (kk / 4) * 64 + (kk % 4) * 8;
            mma_bf16_ts(tmem + 256, tmem + acol, sdesc_sw128_mn(do_addr + kk * 2048, CHUNK),
                        idesc_o, (it > 0 || kk > 0) ? 1u : 0u);
            mma_bf16_ts(tmem + 384, tmem + 128 + acol, sdesc_sw128_mn(q_addr + kk * 2048, CHUNK),
                        idesc_o, (it > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(&r_empty[slot]);
        }
        __syncwarp();
        if (++slot == KV_RING) { slot = 0; ph ^= 1; }
      }
      if (elect_one()) mma_commit(acc_done);
      __syncwarp();
    }
  } else {
    reg_alloc<200>();
    const int hf = (warp - 4) >> 2;     // query half of the tile
    const int ew = (warp - 4) & 3;
    const int r = ew * 32 + lane_id();  // key row in the tile
    const int k = k0 + r;
    const bool row_ok = k < a.L;
    const uint32_t lane_off = static_cast<uint32_t>(ew * 32) << 16;
    const float sl2 = a.scale_log2;
    // queries that see key k: [k, q_vis_end)
    const int q_vis_end = !row_ok ? 0 : k < a.Lp ? a.L : min(a.L, a.Lp + (seg_of(k, m) + 1) * a.Lmax);
    int slot = 0, it = 0;
    uint32_t ph = 0;
    int hh, qt;
    for (int i = 0; next(i, hh, qt); ++i, ++it) {
      mbar_wait(&r_full[slot], ph);  // this stage's lse / D have landed
      const float* st_lse = reinterpret_cast<const float*>(smem + KV_OFF_RING + slot * KV_STAGE + 2 * TILE);
      const float* st_d = st_lse + 128;
      mbar_wait(s_full, it & 1);
      tc_fence_after();
      uint32_t s0[32], s1[32], d0[32], d1[32];
      tmem_ld32(tmem + lane_off + hf * 64, s0);
      tmem_ld32(tmem + lane_off + hf * 64 + 32, s1);
      tmem_ld32(tmem + lane_off + 128 + hf * 64, d0);
      tmem_ld32(tmem + lane_off + 128 + hf * 64 + 32, d1);
      tmem_ld_wait();
      const int qb = qt * TQ + hf * 64;
      // visible query columns: k <= q < q_vis_end
      const uint32_t vis0 = lt_bits(q_vis_end, qb) & ~lt_bits(k, qb);
      const uint32_t vis1 = lt_bits(q_vis_end, qb + 32) & ~lt_bits(k, qb + 32);
      uint32_t wp[32], wd[32];
#pragma unroll
      for (int i2 = 0; i2 < 16; ++i2) {
        float p[4], g[4];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int j = 2 * i2 + e;
          const int c0 = hf * 64 + j, c1 = c0 + 32;
          p[e] = ((vis0 >> j) & 1u) ? exp2_mufu(__uint_as_float(s0[j]) * sl2 - st_lse[c0]) : 0.f;
          p[2 + e] = ((vis1 >> j) & 1u) ? exp2_mufu(__uint_as_float(s1[j]) * sl2 - st_lse[c1]) : 0.f;
          g[e] = p[e] * (__uint_as_float(d0[j]) - st_d[c0]);
          g[2 + e] = p[2 + e] * (__uint_as_float(d1[j]) - st_d[c1]);
        }
        wp[i2] = pack_bf16(p[0], p[1]);
        wp[16 + i2] = pack_bf16(p[2], p[3]);
        wd[i2] = pack_bf16(g[0], g[1]);
        wd[16 + i2] = pack_bf16(g[2], g[3]);
      }
      tmem_st32(tmem + lane_off + hf * 64, wp);
      tmem_st32(tmem + lane_off + 128 + hf * 64, wd);
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(ds_full);
      if (++slot == KV_RING) { slot = 0; ph ^= 1; }
    }
    // epilogue: warpgroup 0 writes dV, warpgroup 1 dK (scaled)
    const int col0 = (hf ? a.k_col0 : a.v_col0) + kvh * HD;
    const float mul = hf ? a.scale : 1.0f;
    __nv_bfloat16* out = a.dqkv + static_cast<size_t>(k) * a.ld_dqkv + col0;
    if (it > 0) {
      mbar_wait(acc_done, 0);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < HD; c += 32) {
        uint32_t o[32];
        tmem_ld32(tmem + lane_off + 256 + hf * 128 + c, o);
        tmem_ld_wait();
        if (row_ok) {
          uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 16; ++j)
            pk[j] = pack_bf16(__uint_as_float(o[2 * j]) * mul, __uint_as_float(o[2 * j + 1]) * mul);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            reinterpret_cast<uint4*>(out + c)[j] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
        }
      }
    } else if (row_ok) {
      for (int c = 0; c < HD; c += 8) *reinterpret_cast<uint4*>(out + c) = make_uint4(0, 0, 0, 0);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// ----------------------------------------------------------------------------
// v2: the same two kernels with the S / dP work split into 64-wide halves and
// TWO TMEM buffers, so the tensor core computes the next half's S and dP (and
// the previous half's accumulator MMAs) while the softmax warps turn this
// half's S, dP into P, dS — v1 leaves the tensor pipe idle during every
// softmax (41-44% busy under ncu). TMEM = [S_0 | dP_0] [S_1 | dP_1] (64 + 64
// columns each) | two 128-column accumulators. The 64-wide S / dP MMAs
// (M 128, N 64, both operands in smem) run at 2/3 rate (smem bandwidth); the
// accumulator MMAs take A from TMEM at full rate.
constexpr int H_CHUNK = 64 * 64 * 2;  // 64 rows x 64 bf16 columns, SW128 (8 KB)
constexpr int HALF = 2 * H_CHUNK;     // 64 x 128 bf16 (16 KB)

__device__ __forceinline__ uint32_t half_kmajor_off(int kk) { return (kk / 4) * H_CHUNK + (kk % 4) * 32; }

// Does any query of [q0, q0 + nq) see any key of [k0, k0 + nk)? (superset test;
// the softmax warps apply the exact per-element mask)
__device__ __forceinline__ bool range_visible(int q0, int nq, int k0, int nk, const MaskDev& m) {
  const int q1 = min(q0 + nq - 1, m.L - 1), k1 = min(k0 + nk - 1, m.L - 1);
  if (q0 >= m.L || k0 >= m.L || k0 > q1) return false;
  if (k0 < m.Lp) return true;  // a prefix key: seen by every later query
  if (q1 < m.Lp) return false;
  const int sk0 = seg_of(k0, m), sk1 = seg_of(k1, m);
  const int qs0 = seg_of(max(q0, m.Lp), m), qs1 = seg_of(q1, m);
  return sk1 >= qs0 && sk0 <= qs1;
}

// A 128 x 64 bf16 half row of a constant A operand (this thread's row) into
// 32 packed TMEM columns (lane = row, column c = elements 2c, 2c + 1).
__device__ __forceinline__ void operand_row_to_tmem(const __nv_bfloat16* row, bool ok, uint32_t taddr) {
  const uint4* src = reinterpret_cast<const uint4*>(row);
  uint32_t w[32];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint4 x = ok ? __ldg(src + j) : make_uint4(0, 0, 0, 0);
    w[4 * j] = x.x; w[4 * j + 1] = x.y; w[4 * j + 2] = x.z; w[4 * j + 3] = x.w;
  }
  tmem_st32(taddr, w);
}

// dK / dV out of TMEM (dV at column 256, dK at 384; warpgroup hf = 0 writes dV,
// 1 writes dK scaled): bf16 into dqkv, or the fp32 partials of a shared kv head.
__device__ __forceinline__ void dkdv_epilogue(const BwdArgs& a, uint32_t tmem, uint32_t lane_off, int hf, int k,
                                              bool row_ok, int kvh, int it, uint64_t* acc_done) {
  const int col0 = (hf ? a.k_col0 : a.v_col0) + kvh * HD;
  const float mul = hf ? a.scale : 1.0f;
  __nv_bfloat16* out = a.dqkv + static_cast<size_t>(k) * a.ld_dqkv + col0;
  if (a.dkv32 != nullptr) {  // fp32 partials (a kv head shared by several ranks)
    const int n_kv_local = a.n_heads / a.q_per_kv;
    float* o32 = a.dkv32 + static_cast<size_t>(k) * a.ld_dkv32 + ((hf ? 0 : n_kv_local) + kvh) * HD;
    if (it > 0) {
      mbar_wait(acc_done, 0);
      tc_fence_after();
    }
#pragma unroll 1
    for (int c = 0; c < HD; c += 32) {
      uint32_t o[32];
      if (it > 0) {
        tmem_ld32(tmem + lane_off + 256 + hf * 128 + c, o);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) o[j] = 0u;
      }
      if (row_ok) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          reinterpret_cast<float4*>(o32 + c)[j] =
              make_float4(__uint_as_float(o[4 * j]) * mul, __uint_as_float(o[4 * j + 1]) * mul,
                          __uint_as_float(o[4 * j + 2]) * mul, __uint_as_float(o[4 * j + 3]) * mul);
      }
    }
  } else if (it > 0) {
    mbar_wait(acc_done, 0);
    tc_fence_after();
#pragma unroll 1
    for (int c = 0; c < HD; c += 32) {
      uint32_t o[32];
      tmem_ld32(tmem + lane_off + 256 + hf * 128 + c, o);
      tmem_ld_wait();
      if (row_ok) {
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j)
          pk[j] = pack_bf16(__uint_as_float(o[2 * j]) * mul, __uint_as_float(o[2 * j + 1]) * mul);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          reinterpret_cast<uint4*>(out + c)[j] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
      }
    }
  } else if (row_ok) {
    for (int c = 0; c < HD; c += 8) *reinterpret_cast<uint4*>(out + c) = make_uint4(0, 0, 0, 0);
  }
}

// dK, dV (v2): one CTA per (key tile, kv head); items = (64-query half block,
// query head of the group).
constexpr int KV2_RING = 4;
constexpr int KV2_STAT = 2 * 64 * 4;
constexpr int KV2_STAGE = (2 * HALF + KV2_STAT + 1023) / 1024 * 1024;
constexpr int KV2_OFF_K = 0, KV2_OFF_V = TILE, KV2_OFF_RING = 2 * TILE;
constexpr int KV2_OFF_BAR = KV2_OFF_RING + KV2_RING * KV2_STAGE;
constexpr size_t KV2_SMEM = 1024 + KV2_OFF_BAR + 256;

__global__ void __launch_bounds__(THREADS, 1)
    attn_bwd_dkdv2(const __grid_constant__ CUtensorMap tmQKV, const __grid_constant__ CUtensorMap tmQ64,
                   const __grid_constant__ CUtensorMap tmDO64, const __grid_constant__ CUtensorMap tmLSE,
                   const __grid_constant__ CUtensorMap tmD, BwdArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + KV2_OFF_BAR);
  uint64_t* kv_full = bars;
  uint64_t* r_full = bars + 1;              // [KV2_RING]
  uint64_t* r_empty = bars + 1 + KV2_RING;  // [KV2_RING]
  uint64_t* s_full = bars + 1 + 2 * KV2_RING;  // [2] per TMEM buffer
  uint64_t* ds_full = s_full + 2;              // [2]
  uint64_t* acc_done = s_full + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 5);

  const int warp = warp_id();
  BTRACE_INIT(0);
  const MaskDev m = mask_of(a);
  const int n_kt = (a.L + TK - 1) / TK;
  const int kvh = blockIdx.x / n_kt;
  const int kt = blockIdx.x - kvh * n_kt;
  const int k0 = kt * TK;
  const int q_end = k0 < a.Lp ? a.L : min(a.L, a.Lp + (seg_of(min(k0 + TK - 1, a.L - 1), m) + 1) * a.Lmax);
  const int qb_lo = k0 / 64, qb_hi = (q_end + 63) / 64;
  // Items (64-row query block, query head of the group), head-minor. Every
  // block in [qb_lo, qb_hi) sees the key tile (prefix keys: every later query;
  // row keys: the queries of their rows' segments, contiguous up to q_end), so
  // the walk only skips the blocks of other row parts — incrementally, no
  // per-item divisions (every role of every thread repeats it).
  struct Items {
    int qb, hh;
    __device__ void own(const BwdArgs& a, int hi) {
      while (qb < hi && !own_rows(qb * 64, a)) ++qb;
    }
  };
  auto items_begin = [&]() {
    Items t{qb_lo, 0};
    t.own(a, qb_hi);
    return t;
  };
  auto items_next = [&](Items& t) {
    if (++t.hh == a.q_per_kv) {
      t.hh = 0;
      ++t.qb;
      t.own(a, qb_hi);
    }
  };

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmQKV);
    tma_prefetch_desc(&tmQ64);
    tma_prefetch_desc(&tmDO64);
    tma_prefetch_desc(&tmLSE);
    tma_prefetch_desc(&tmD);
    mbar_init(kv_full, 1);
    for (int s = 0; s < KV2_RING; ++s) {
      mbar_init(&r_full[s], 1);
      mbar_init(&r_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&ds_full[b], 256);
    }
    mbar_init(acc_done, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    reg_dealloc<56>();
    if (warp == 0) {
      if (elect_one()) {
        mbar_arrive_expect_tx(kv_full, 2 * TILE);
        for (int c = 0; c < 2; ++c) {
          tma_load_2d(smem + KV2_OFF_K + c * CHUNK, &tmQKV, kv_full, a.k_col0 + kvh * HD + c * 64, k0);
          tma_load_2d(smem + KV2_OFF_V + c * CHUNK, &tmQKV, kv_full, a.v_col0 + kvh * HD + c * 64, k0);
        }
        int slot = 0;
        uint32_t ph = 0;
        for (Items t = items_begin(); t.qb < qb_hi; items_next(t)) {
          const int qb = t.qb, h = kvh * a.q_per_kv + t.hh;
          mbar_wait(&r_empty[slot], ph ^ 1);
          BTRACE(20, qb);
          mbar_arrive_expect_tx(&r_full[slot], 2 * HALF + KV2_STAT);
          uint8_t* st = smem + KV2_OFF_RING + slot * KV2_STAGE;
          for (int c = 0; c < 2; ++c) {
            tma_load_2d(st + c * H_CHUNK, &tmQ64, &r_full[slot], a.q_col0 + h * HD + c * 64, qb * 64);
            tma_load_2d(st + HALF + c * H_CHUNK, &tmDO64, &r_full[slot], h * HD + c * 64, qb * 64);
          }
          tma_load_2d(st + 2 * HALF, &tmLSE, &r_full[slot], qb * 64, h);
          tma_load_2d(st + 2 * HALF + 256, &tmD, &r_full[slot], qb * 64, h);
          if (++slot == KV2_RING) { slot = 0; ph ^= 1; }
        }
      }
    } else if (warp == 1) {
      const uint32_t idesc_s = idesc_bf16_f32(TK, 64);
      const uint32_t idesc_o = idesc_bf16_f32_bmn(TK, HD);
      const uint32_t k_addr = smem_u32(smem + KV2_OFF_K), v_addr = smem_u32(smem + KV2_OFF_V);
      const uint32_t ring = smem_u32(smem + KV2_OFF_RING);
      mbar_wait(kv_full, 0);
      auto issue_sdp = [&](int it, int slot) {
        const uint32_t tb = tmem + (it & 1) * 128;
        const uint32_t q_addr = ring + slot * KV2_STAGE, do_addr = q_addr + HALF;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk)
            mma_bf16_ss(tb, sdesc_sw128(k_addr + kmajor_off(kk)), sdesc_sw128(q_addr + half_kmajor_off(kk)),
                        idesc_s, kk > 0 ? 1u : 0u);
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk)
            mma_bf16_ss(tb + 64, sdesc_sw128(v_addr + kmajor_off(kk)),
                        sdesc_sw128(do_addr + half_kmajor_off(kk)), idesc_s, kk > 0 ? 1u : 0u);
          mma_commit(&s_full[it & 1]);
        }
        __syncwarp();
      };
      auto issue_acc = [&](int it, int slot) {
        mbar_wait(&ds_full[it & 1], (it >> 1) & 1);
        BTRACE(12, it);
        tc_fence_after();
        const uint32_t q_addr = ring + slot * KV2_STAGE, do_addr = q_addr + HALF;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 64 / 16; ++kk) {
            const uint32_t acol = (it & 1) * 128 + (kk / 2) * 32 + (kk % 2) * 8;
            mma_bf16_ts(tmem + 256, tmem + acol, sdesc_sw128_mn(do_addr + kk * 2048, H_CHUNK),
                        idesc_o, (it > 0 || kk > 0) ? 1u : 0u);
            mma_bf16_ts(tmem + 384, tmem + 64 + acol, sdesc_sw128_mn(q_addr + kk * 2048, H_CHUNK),
                        idesc_o, (it > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(&r_empty[slot]);
        }
        __syncwarp();
      };
      int slot = 0, prev = -1, it = 0;
      uint32_t ph = 0;
      for (Items t = items_begin(); t.qb < qb_hi; items_next(t), ++it) {
        mbar_wait(&r_full[slot], ph);
        BTRACE(10, it);
        tc_fence_after();
        issue_sdp(it, slot);
        BTRACE(11, it);
        if (it > 0) issue_acc(it - 1, prev);
        if (it > 0) BTRACE(13, it - 1);
        prev = slot;
        if (++slot == KV2_RING) { slot = 0; ph ^= 1; }
      }
      if (it > 0) issue_acc(it - 1, prev);
      if (elect_one()) mma_commit(acc_done);
      __syncwarp();
    }
  } else {
    reg_alloc<200>();
    const int hf = (warp - 4) >> 2;
    const int ew = (warp - 4) & 3;
    const int r = ew * 32 + lane_id();
    const int k = k0 + r;
    const bool row_ok = k < a.L;
    const uint32_t lane_off = static_cast<uint32_t>(ew * 32) << 16;
    const float sl2 = a.scale_log2;
    const int q_vis_end = !row_ok ? 0 : k < a.Lp ? a.L : min(a.L, a.Lp + (seg_of(k, m) + 1) * a.Lmax);
    int slot = 0, it = 0;
    uint32_t ph = 0;
    for (Items t = items_begin(); t.qb < qb_hi; items_next(t), ++it) {
      const int qb = t.qb;
      mbar_wait(&r_full[slot], ph);
      const float* st_lse = reinterpret_cast<const float*>(smem + KV2_OFF_RING + slot * KV2_STAGE + 2 * HALF);
      const float* st_d = st_lse + 64;
      // this half's 32 lse and D values (broadcast 16-byte shared loads)
      float lse_r[32], d_r[32];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float4 x = reinterpret_cast<const float4*>(st_lse + hf * 32)[j];
        const float4 y = reinterpret_cast<const float4*>(st_d + hf * 32)[j];
        lse_r[4 * j] = x.x; lse_r[4 * j + 1] = x.y; lse_r[4 * j + 2] = x.z; lse_r[4 * j + 3] = x.w;
        d_r[4 * j] = y.x; d_r[4 * j + 1] = y.y; d_r[4 * j + 2] = y.z; d_r[4 * j + 3] = y.w;
      }
      const uint32_t tb = tmem + lane_off + (it & 1) * 128;
      BTRACE(0, it);
      mbar_wait(&s_full[it & 1], (it >> 1) & 1);
      BTRACE(1, it);
      tc_fence_after();
      uint32_t sv[32], dv[32];
      tmem_ld32(tb + hf * 32, sv);
      tmem_ld32(tb + 64 + hf * 32, dv);
      tmem_ld_wait();
      BTRACE(2, it);
      const int qbase = qb * 64 + hf * 32;
      const uint32_t vis = lt_bits(q_vis_end, qbase) & ~lt_bits(k, qbase);
      uint32_t wp[16], wd[16];
#pragma unroll
      for (int j2 = 0; j2 < 16; ++j2) {
        float p[2], g[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int j = 2 * j2 + e;
          p[e] = ((vis >> j) & 1u) ? exp2_mufu(__uint_as_float(sv[j]) * sl2 - lse_r[j]) : 0.f;
          g[e] = p[e] * (__uint_as_float(dv[j]) - d_r[j]);
        }
        wp[j2] = pack_bf16(p[0], p[1]);
        wd[j2] = pack_bf16(g[0], g[1]);
      }
      BTRACE(3, it);
      tmem_st16(tb + hf * 32, wp);
      tmem_st16(tb + 64 + hf * 32, wd);
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&ds_full[it & 1]);
      BTRACE(4, it);
      if (++slot == KV2_RING) { slot = 0; ph ^= 1; }
    }
    dkdv_epilogue(a, tmem, lane_off, hf, k, row_ok, kvh, it, acc_done);
  }
  BTRACE_FINISH;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// dK, dV (v4): 128-query items, ONE S^T / dP^T buffer pair, and the softmax
// handing P^T and dS^T over separately. The tensor core runs, per item i,
//   S^T(i) -> dK += dS^T(i-1) Q(i-1) -> dP^T(i) -> dV += P^T(i) dO(i)
// so the softmax turns S^T(i) into P^T(i) behind dK(i-1) and dP^T(i), and
// dP^T(i) into dS^T(i) behind dV(i) and S^T(i+1). The N = 128 S^T / dP^T MMAs
// read K / V once per 128 queries at the full ss rate (v2's N = 64 halves
// re-read the key tile for every 64 queries and are shared-memory bound,
// profiles/r1_attention_study.md §7b). TMEM = S^T | dP^T | dV | dK (512
// columns), like v1, which handed P^T and dS^T over together after both MMAs
// and so serialised the softmax and the tensor core. P^T goes over in two
// 32-query chunks per warpgroup, so dV starts on the first while the second is
// exponentiated. Each ring stage has two barriers: Q + lse (for S^T and P^T)
// and dO + D (for dP^T and dS^T).
// kPoly: pairs (of every 32) whose exp2 runs on the FMA pipe (P^T is the
// MUFU-bound step on the S^T -> P^T -> dV chain).
// v4 shared memory: K | V, then a 3-deep Q ring and a 2-deep dO ring (Q(i) is
// read by S^T(i) and by dK(i), which runs after S^T(i+1), so three Q tiles
// keep the next load ahead), their lse / D rows, and the barriers: 232,192
// bytes, i.e. no room for the usual 1 KB alignment slack — the kernel traps if
// the dynamic shared window is not 1024-aligned.
constexpr int V4_QR = 3, V4_DR = 2;
constexpr int V4_OFF_K = 0, V4_OFF_V = TILE, V4_OFF_Q = 2 * TILE, V4_OFF_DO = V4_OFF_Q + V4_QR * TILE;
constexpr int V4_OFF_LSE = V4_OFF_DO + V4_DR * TILE, V4_OFF_D = V4_OFF_LSE + V4_QR * 512;
constexpr int V4_OFF_BAR = V4_OFF_D + V4_DR * 512;
constexpr size_t V4_SMEM = V4_OFF_BAR + 256;
static_assert(V4_SMEM <= 232448, "v4 dK / dV shared memory");

template <int kPoly>
__global__ void __launch_bounds__(THREADS, 1)
    attn_bwd_dkdv4(const __grid_constant__ CUtensorMap tmQKV, const __grid_constant__ CUtensorMap tmDO,
                   const __grid_constant__ CUtensorMap tmLSE, const __grid_constant__ CUtensorMap tmD,
                   BwdArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if (smem_u32(smem) & 1023u) __trap();  // the layout has no alignment slack
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + V4_OFF_BAR);
  uint64_t* kv_full = bars;
  uint64_t* rq_full = bars + 1;                    // [V4_QR] Q + lse landed
  uint64_t* rq_empty = rq_full + V4_QR;            // [V4_QR] Q read by S^T and dK
  uint64_t* rd_full = rq_empty + V4_QR;            // [V4_DR] dO + D landed
  uint64_t* rd_empty = rd_full + V4_DR;            // [V4_DR] dO read by dP^T and dV
  uint64_t* s_full = rd_empty + V4_DR;
  uint64_t* dp_full = s_full + 1;
  uint64_t* p_ready = s_full + 2;  // [2]: query columns [32 c, 32 c + 32) of each half
  uint64_t* ds_ready = s_full + 4;
  uint64_t* acc_done = s_full + 5;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 6);

  const int warp = warp_id();
  BTRACE_INIT(0);
  const MaskDev m = mask_of(a);
  const int n_kt = (a.L + TK - 1) / TK;
  const int kvh = blockIdx.x / n_kt;
  const int kt = blockIdx.x - kvh * n_kt;
  const int k0 = kt * TK;
  const int q_end = k0 < a.Lp ? a.L : min(a.L, a.Lp + (seg_of(min(k0 + TK - 1, a.L - 1), m) + 1) * a.Lmax);
  const int qt_lo = k0 / TQ, qt_hi = (q_end + TQ - 1) / TQ;
  struct Items {  // (128-row query tile, query head of the group), head-minor
    int qt, hh;
    __device__ void own(const BwdArgs& a, int hi) {
      while (qt < hi && !own_rows(qt * TQ, a)) ++qt;
    }
  };
  auto items_begin = [&]() {
    Items t{qt_lo, 0};
    t.own(a, qt_hi);
    return t;
  };
  auto items_next = [&](Items& t) {
    if (++t.hh == a.q_per_kv) {
      t.hh = 0;
      ++t.qt;
      t.own(a, qt_hi);
    }
  };

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmQKV);
    tma_prefetch_desc(&tmDO);
    tma_prefetch_desc(&tmLSE);
    tma_prefetch_desc(&tmD);
    mbar_init(kv_full, 1);
    for (int s = 0; s < V4_QR; ++s) {
      mbar_init(&rq_full[s], 1);
      mbar_init(&rq_empty[s], 1);
    }
    for (int s = 0; s < V4_DR; ++s) {
      mbar_init(&rd_full[s], 1);
      mbar_init(&rd_empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(dp_full, 1);
    mbar_init(&p_ready[0], 256);
    mbar_init(&p_ready[1], 256);
    mbar_init(ds_ready, 256);
    mbar_init(acc_done, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;  // S^T [0,128) dP^T [128,256) dV [256,384) dK [384,512)

  if (warp < 4) {
    reg_dealloc<56>();
    if (warp == 0) {
      if (elect_one()) {
        mbar_arrive_expect_tx(kv_full, 2 * TILE);
        for (int c = 0; c < 2; ++c) {
          tma_load_2d(smem + V4_OFF_K + c * CHUNK, &tmQKV, kv_full, a.k_col0 + kvh * HD + c * 64, k0);
          tma_load_2d(smem + V4_OFF_V + c * CHUNK, &tmQKV, kv_full, a.v_col0 + kvh * HD + c * 64, k0);
        }
        int qs = 0, ds = 0;
        uint32_t qph = 0, dph = 0;
        for (Items t = items_begin(); t.qt < qt_hi; items_next(t)) {
          const int qt = t.qt, h = kvh * a.q_per_kv + t.hh;
          mbar_wait(&rq_empty[qs], qph ^ 1);
          BTRACE(20, qt);
          mbar_arrive_expect_tx(&rq_full[qs], TILE + 512);
          for (int c = 0; c < 2; ++c)
            tma_load_2d(smem + V4_OFF_Q + qs * TILE + c * CHUNK, &tmQKV, &rq_full[qs],
                        a.q_col0 + h * HD + c * 64, qt * TQ);
          tma_load_2d(smem + V4_OFF_LSE + qs * 512, &tmLSE, &rq_full[qs], qt * TQ, h);
          mbar_wait(&rd_empty[ds], dph ^ 1);
          mbar_arrive_expect_tx(&rd_full[ds], TILE + 512);
          for (int c = 0; c < 2; ++c)
            tma_load_2d(smem + V4_OFF_DO + ds * TILE + c * CHUNK, &tmDO, &rd_full[ds], h * HD + c * 64,
                        qt * TQ);
          tma_load_2d(smem + V4_OFF_D + ds * 512, &tmD, &rd_full[ds], qt * TQ, h);
          if (++qs == V4_QR) { qs = 0; qph ^= 1; }
          if (++ds == V4_DR) { ds = 0; dph ^= 1; }
        }
      }
    } else if (warp == 1) {
      const uint32_t idesc_s = idesc_bf16_f32(TK, TQ);
      const uint32_t idesc_o = idesc_bf16_f32_bmn(TK, HD);
      const uint32_t k_addr = smem_u32(smem + V4_OFF_K), v_addr = smem_u32(smem + V4_OFF_V);
      const uint32_t qring = smem_u32(smem + V4_OFF_Q), dring = smem_u32(smem + V4_OFF_DO);
      mbar_wait(kv_full, 0);
      // dK += dS^T(j) Q(j) (A: packed pairs in columns [128,160) + [192,224)),
      // then the ring slot of item j is free
      auto issue_dk = [&](int j, int jslot) {
        mbar_wait(ds_ready, j & 1);
        BTRACE(14, j);
        tc_fence_after();
        const uint32_t q_addr = qring + jslot * TILE;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < TQ / 16; ++kk)
            mma_bf16_ts(tmem + 384, tmem + 128 + (kk / 4) * 64 + (kk % 4) * 8,
                        sdesc_sw128_mn(q_addr + kk * 2048, CHUNK), idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
          mma_commit(&rq_empty[jslot]);
        }
        __syncwarp();
      };
      int qs = 0, ds = 0, prev = 0, it = 0;
      uint32_t qph = 0, dph = 0;
      for (Items t = items_begin(); t.qt < qt_hi; items_next(t), ++it) {
        const uint32_t q_addr = qring + qs * TILE, do_addr = dring + ds * TILE;
        // S^T(i) overwrites P^T(i-1) and dP^T(i) overwrites dS^T(i-1): both
        // read by MMAs issued earlier, and the tensor pipe runs in issue order
        mbar_wait(&rq_full[qs], qph);
        BTRACE(10, it);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk)
            mma_bf16_ss(tmem, sdesc_sw128(k_addr + kmajor_off(kk)), sdesc_sw128(q_addr + kmajor_off(kk)),
                        idesc_s, kk > 0 ? 1u : 0u);
          mma_commit(s_full);
        }
        __syncwarp();
        if (it > 0) issue_dk(it - 1, prev);
        mbar_wait(&rd_full[ds], dph);
        BTRACE(11, it);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk)
            mma_bf16_ss(tmem + 128, sdesc_sw128(v_addr + kmajor_off(kk)),
                        sdesc_sw128(do_addr + kmajor_off(kk)), idesc_s, kk > 0 ? 1u : 0u);
          mma_commit(dp_full);
        }
        __syncwarp();
        // dV += P^T(i) dO(i) (A: packed pairs in columns [0,32) + [64,96)), in
        // the two chunks the softmax hands over: K steps {0,1,4,5}, {2,3,6,7}
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          mbar_wait(&p_ready[c], it & 1);
          if (c == 0) BTRACE(12, it);
          tc_fence_after();
          if (elect_one()) {
#pragma unroll
            for (int k4 = 0; k4 < 4; ++k4) {
              const int kk = (k4 >> 1) * 4 + c * 2 + (k4 & 1);
              mma_bf16_ts(tmem + 256, tmem + (kk / 4) * 64 + (kk % 4) * 8,
                          sdesc_sw128_mn(do_addr + kk * 2048, CHUNK), idesc_o, (it > 0 || kk > 0) ? 1u : 0u);
            }
          }
          __syncwarp();
        }
        if (elect_one()) mma_commit(&rd_empty[ds]);  // dO(i) read by dP^T(i) and dV(i)
        __syncwarp();
        BTRACE(13, it);
        prev = qs;
        if (++qs == V4_QR) { qs = 0; qph ^= 1; }
        if (++ds == V4_DR) { ds = 0; dph ^= 1; }
      }
      if (it > 0) issue_dk(it - 1, prev);
      if (elect_one()) mma_commit(acc_done);
      __syncwarp();
    }
  } else {
    reg_alloc<200>();
    const int hf = (warp - 4) >> 2;  // query columns [64 hf, 64 hf + 64) of the item
    const int ew = (warp - 4) & 3;
    const int r = ew * 32 + lane_id();
    const int k = k0 + r;
    const bool row_ok = k < a.L;
    const uint32_t lane_off = static_cast<uint32_t>(ew * 32) << 16;
    const float sl2 = a.scale_log2;
    const int q_vis_end = !row_ok ? 0 : k < a.Lp ? a.L : min(a.L, a.Lp + (seg_of(k, m) + 1) * a.Lmax);
    const uint32_t tS = tmem + lane_off + hf * 64, tP = tmem + lane_off + 128 + hf * 64;
    int qs = 0, ds = 0, it = 0;
    uint32_t qph = 0, dph = 0;
    for (Items t = items_begin(); t.qt < qt_hi; items_next(t), ++it) {
      const int qbase = t.qt * TQ + hf * 64;
      const float4* st_lse = reinterpret_cast<const float4*>(smem + V4_OFF_LSE + qs * 512) + hf * 16;
      const float4* st_d = reinterpret_cast<const float4*>(smem + V4_OFF_D + ds * 512) + hf * 16;
      float p[64];
      mbar_wait(&rq_full[qs], qph);
      BTRACE(0, it);
      mbar_wait(s_full, it & 1);
      BTRACE(1, it);
      tc_fence_after();
      uint32_t w[32];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t sv[32], wc[16];
        tmem_ld32(tS + c * 32, sv);
        tmem_ld_wait();
        const uint32_t vis = lt_bits(q_vis_end, qbase + 32 * c) & ~lt_bits(k, qbase + 32 * c);
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
          const float4 l4 = st_lse[c * 8 + j4];
          float x[4];
          ffma2(x[0], x[1], __uint_as_float(sv[4 * j4]), __uint_as_float(sv[4 * j4 + 1]), sl2, sl2, -l4.x,
                -l4.y);
          ffma2(x[2], x[3], __uint_as_float(sv[4 * j4 + 2]), __uint_as_float(sv[4 * j4 + 3]), sl2, sl2, -l4.z,
                -l4.w);
#pragma unroll
          for (int e = 0; e < 4; e += 2) {
            const int j = 4 * j4 + e;
            float y0, y1;
            if (poly_pair<kPoly>(16 * c + j / 2)) {
              exp2_poly2(x[e], x[e + 1], y0, y1);
            } else {
              y0 = exp2_mufu(x[e]);
              y1 = exp2_mufu(x[e + 1]);
            }
            p[32 * c + j] = ((vis >> j) & 1u) ? y0 : 0.f;
            p[32 * c + j + 1] = ((vis >> (j + 1)) & 1u) ? y1 : 0.f;
          }
          wc[2 * j4] = pack_bf16(p[32 * c + 4 * j4], p[32 * c + 4 * j4 + 1]);
          wc[2 * j4 + 1] = pack_bf16(p[32 * c + 4 * j4 + 2], p[32 * c + 4 * j4 + 3]);
        }
        // packed P^T of these 32 queries over columns [16 c, 16 c + 16) of the
        // half (S^T of chunk 0 is consumed; chunk 1's S^T lies in [32, 64))
        tmem_st16(tS + 16 * c, wc);
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&p_ready[c]);
      }
      BTRACE(3, it);
      mbar_wait(&rd_full[ds], dph);
      mbar_wait(dp_full, it & 1);
      BTRACE(4, it);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t dv[32];
        tmem_ld32(tP + c * 32, dv);
        tmem_ld_wait();
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
          const float4 d4 = st_d[c * 8 + j4];
          float g[4];
          fsub2(g[0], g[1], __uint_as_float(dv[4 * j4]), __uint_as_float(dv[4 * j4 + 1]), d4.x, d4.y);
          fsub2(g[2], g[3], __uint_as_float(dv[4 * j4 + 2]), __uint_as_float(dv[4 * j4 + 3]), d4.z, d4.w);
          fmul2(g[0], g[1], p[32 * c + 4 * j4], p[32 * c + 4 * j4 + 1], g[0], g[1]);
          fmul2(g[2], g[3], p[32 * c + 4 * j4 + 2], p[32 * c + 4 * j4 + 3], g[2], g[3]);
          w[16 * c + 2 * j4] = pack_bf16(g[0], g[1]);
          w[16 * c + 2 * j4 + 1] = pack_bf16(g[2], g[3]);
        }
      }
      tmem_st32(tP, w);  // packed dS^T
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(ds_ready);
      BTRACE(5, it);
      if (++qs == V4_QR) { qs = 0; qph ^= 1; }
      if (++ds == V4_DR) { ds = 0; dph ^= 1; }
    }
    dkdv_epilogue(a, tmem, lane_off, hf, k, row_ok, kvh, it, acc_done);
  }
  BTRACE_FINISH;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// dQ (v2): one CTA per (query tile, query head); items = 64-key half tiles.
// kTmemA: Q and dO, the A operands of every S / dP MMA of the CTA, live in
// TMEM (columns 384 | 448, packed bf16, written once by the softmax warps), so
// the 64-wide S / dP MMAs read only B from shared memory and run at full rate
// instead of the 2/3 of the smem-bound ss form. TMEM = [S_0|dP_0] [S_1|dP_1]
// | dQ | Q | dO = 512 columns.
constexpr int DQ2_RING = 4;  // K half | V half per stage
constexpr int DQ2_STAGE = 2 * HALF;
constexpr int DQ2_OFF_Q = 0, DQ2_OFF_DO = TILE, DQ2_OFF_RING = 2 * TILE;
constexpr int DQ2_OFF_BAR = DQ2_OFF_RING + DQ2_RING * DQ2_STAGE;
constexpr size_t DQ2_SMEM = 1024 + DQ2_OFF_BAR + 256;

// kPoly: pairs (of every 32) whose exp2 runs on the FMA pipe.
template <bool kTmemA, int kPoly = 0>
__global__ void __launch_bounds__(THREADS, 1)
    attn_bwd_dq2(const __grid_constant__ CUtensorMap tmQKV, const __grid_constant__ CUtensorMap tmKV64,
                 const __grid_constant__ CUtensorMap tmDO, BwdArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + DQ2_OFF_BAR);
  uint64_t* q_full = bars;
  uint64_t* r_full = bars + 1;
  uint64_t* r_empty = bars + 1 + DQ2_RING;
  uint64_t* s_full = bars + 1 + 2 * DQ2_RING;  // [2]
  uint64_t* ds_full = s_full + 2;              // [2]
  uint64_t* dq_done = s_full + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 5);

  const int warp = warp_id();
  BTRACE_INIT(1);
  const MaskDev m = mask_of(a);
  const int n_qt = (a.L + TQ - 1) / TQ;
  const int n_tiles = a.row_parts > 1 ? 2 * a.n_local_blocks : n_qt;
  const int per_kv = n_tiles * a.q_per_kv;
  const int kvh = blockIdx.x / per_kv;
  const int rem = blockIdx.x - kvh * per_kv;
  const int qt = dq_tile(rem / a.q_per_kv, a, n_qt);
  const int h = kvh * a.q_per_kv + rem % a.q_per_kv;
  const int q0 = qt * TQ;
  // Keys this query tile sees, as two contiguous 64-key block ranges: the
  // prompt [0, min(Lp, q_last + 1)) and the rows' own segments
  // [segment start of max(q0, Lp), q_last + 1) (empty for a prompt tile)
  const int q_last = min(q0 + TQ - 1, a.L - 1);
  const int r1_hi = (min(a.Lp, q_last + 1) + 63) / 64;
  int r2_lo = r1_hi, r2_hi = r1_hi;
  if (q_last >= a.Lp) {
    const int seg_start = a.Lp + seg_of(max(q0, a.Lp), m) * a.Lmax;
    r2_lo = max(r1_hi, seg_start / 64);
    r2_hi = (q_last + 1 + 63) / 64;
  }
  auto kb_first = [&]() { return r1_hi > 0 ? 0 : r2_lo; };
  auto kb_next = [&](int kb) { return kb + 1 == r1_hi ? r2_lo : kb + 1; };

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmQKV);
    tma_prefetch_desc(&tmKV64);
    tma_prefetch_desc(&tmDO);
    mbar_init(q_full, kTmemA ? 256 : 1);
    for (int s = 0; s < DQ2_RING; ++s) {
      mbar_init(&r_full[s], 1);
      mbar_init(&r_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&ds_full[b], 256);
    }
    mbar_init(dq_done, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    reg_dealloc<56>();
    if (warp == 0) {
      if (elect_one()) {
        if (!kTmemA) {
          mbar_arrive_expect_tx(q_full, 2 * TILE);
          for (int c = 0; c < 2; ++c) {
            tma_load_2d(smem + DQ2_OFF_Q + c * CHUNK, &tmQKV, q_full, a.q_col0 + h * HD + c * 64, q0);
            tma_load_2d(smem + DQ2_OFF_DO + c * CHUNK, &tmDO, q_full, h * HD + c * 64, q0);
          }
        }
        int slot = 0;
        uint32_t ph = 0;
        for (int kb = kb_first(); kb < r2_hi; kb = kb_next(kb)) {
          mbar_wait(&r_empty[slot], ph ^ 1);
          mbar_arrive_expect_tx(&r_full[slot], DQ2_STAGE);
          uint8_t* st = smem + DQ2_OFF_RING + slot * DQ2_STAGE;
          for (int c = 0; c < 2; ++c) {
            tma_load_2d(st + c * H_CHUNK, &tmKV64, &r_full[slot], a.k_col0 + kvh * HD + c * 64, kb * 64);
            tma_load_2d(st + HALF + c * H_CHUNK, &tmKV64, &r_full[slot], a.v_col0 + kvh * HD + c * 64, kb * 64);
          }
          if (++slot == DQ2_RING) { slot = 0; ph ^= 1; }
        }
      }
    } else if (warp == 1) {
      const uint32_t idesc_s = idesc_bf16_f32(TQ, 64);
      const uint32_t idesc_o = idesc_bf16_f32_bmn(TQ, HD);
      const uint32_t q_addr = smem_u32(smem + DQ2_OFF_Q), do_addr = smem_u32(smem + DQ2_OFF_DO);
      const uint32_t ring = smem_u32(smem + DQ2_OFF_RING);
      mbar_wait(q_full, 0);
      tc_fence_after();
      auto issue_sdp = [&](int it, int slot) {
        const uint32_t tb = tmem + (it & 1) * 128;
        const uint32_t kh = ring + slot * DQ2_STAGE, vh = kh + HALF;
        if (elect_one()) {
          if (kTmemA) {
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk)
              mma_bf16_ts(tb, tmem + 384 + kk * 8, sdesc_sw128(kh + half_kmajor_off(kk)), idesc_s,
                          kk > 0 ? 1u : 0u);
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk)
              mma_bf16_ts(tb + 64, tmem + 448 + kk * 8, sdesc_sw128(vh + half_kmajor_off(kk)), idesc_s,
                          kk > 0 ? 1u : 0u);
          } else {
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk)
              mma_bf16_ss(tb, sdesc_sw128(q_addr + kmajor_off(kk)), sdesc_sw128(kh + half_kmajor_off(kk)),
                          idesc_s, kk > 0 ? 1u : 0u);
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk)
              mma_bf16_ss(tb + 64, sdesc_sw128(do_addr + kmajor_off(kk)),
                          sdesc_sw128(vh + half_kmajor_off(kk)), idesc_s, kk > 0 ? 1u : 0u);
          }
          mma_commit(&s_full[it & 1]);
        }
        __syncwarp();
      };
      auto issue_acc = [&](int it, int slot) {
        mbar_wait(&ds_full[it & 1], (it >> 1) & 1);
        BTRACE(12, it);
        tc_fence_after();
        const uint32_t kh = ring + slot * DQ2_STAGE;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 64 / 16; ++kk)
            mma_bf16_ts(tmem + 256, tmem + (it & 1) * 128 + (kk / 2) * 32 + (kk % 2) * 8,
                        sdesc_sw128_mn(kh + kk * 2048, H_CHUNK), idesc_o, (it > 0 || kk > 0) ? 1u : 0u);
          mma_commit(&r_empty[slot]);
        }
        __syncwarp();
      };
      int slot = 0, prev = -1, it = 0;
      uint32_t ph = 0;
      for (int kb = kb_first(); kb < r2_hi; kb = kb_next(kb), ++it) {
        mbar_wait(&r_full[slot], ph);
        BTRACE(10, it);
        tc_fence_after();
        issue_sdp(it, slot);
        BTRACE(11, it);
        if (it > 0) issue_acc(it - 1, prev);
        if (it > 0) BTRACE(13, it - 1);
        prev = slot;
        if (++slot == DQ2_RING) { slot = 0; ph ^= 1; }
      }
      if (it > 0) issue_acc(it - 1, prev);
      if (elect_one()) mma_commit(dq_done);
      __syncwarp();
    }
  } else {
    reg_alloc<200>();
    const int hf = (warp - 4) >> 2;
    const int ew = (warp - 4) & 3;
    const int r = ew * 32 + lane_id();
    const int q = q0 + r;
    const bool row_ok = q < a.L;
    const uint32_t lane_off = static_cast<uint32_t>(ew * 32) << 16;
    const float lse = row_ok ? a.lse[static_cast<size_t>(h) * a.ld_stat + q] : INFINITY;
    const float Dq = row_ok ? a.D[static_cast<size_t>(h) * a.ld_stat + q] : 0.f;
    const float sl2 = a.scale_log2;
    const int k_end = min(q + 1, a.L), k_mid = a.Lp;
    const int k_lo = q >= a.Lp ? a.Lp + seg_of(q, m) * a.Lmax : 0;
    if (kTmemA) {  // this thread's Q / dO row half into the A-operand columns
      const __nv_bfloat16* qrow = a.qkv + static_cast<size_t>(q) * a.ld_qkv + a.q_col0 + h * HD + hf * 64;
      const __nv_bfloat16* drow = a.dO + static_cast<size_t>(q) * a.ld_do + h * HD + hf * 64;
      operand_row_to_tmem(qrow, row_ok, tmem + lane_off + 384 + hf * 32);
      operand_row_to_tmem(drow, row_ok, tmem + lane_off + 448 + hf * 32);
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(q_full);
    }
    int it = 0;
    for (int kb = kb_first(); kb < r2_hi; kb = kb_next(kb), ++it) {
      const uint32_t tb = tmem + lane_off + (it & 1) * 128;
      BTRACE(0, it);
      mbar_wait(&s_full[it & 1], (it >> 1) & 1);
      BTRACE(1, it);
      tc_fence_after();
      uint32_t sv[32], dv[32];
      tmem_ld32(tb + hf * 32, sv);
      tmem_ld32(tb + 64 + hf * 32, dv);
      tmem_ld_wait();
      const int kbase = kb * 64 + hf * 32;
      const uint32_t vis = lt_bits(k_end, kbase) & (lt_bits(k_mid, kbase) | ~lt_bits(k_lo, kbase));
      uint32_t w[16];
#pragma unroll
      for (int j2 = 0; j2 < 16; ++j2) {
        const int j = 2 * j2;
        float x0, x1, y0, y1;
        ffma2(x0, x1, __uint_as_float(sv[j]), __uint_as_float(sv[j + 1]), sl2, sl2, -lse, -lse);
        if (poly_pair<kPoly>(j2 + 16 * hf)) {
          exp2_poly2(x0, x1, y0, y1);
        } else {
          y0 = exp2_mufu(x0);
          y1 = exp2_mufu(x1);
        }
        const float p0 = ((vis >> j) & 1u) ? y0 : 0.f, p1 = ((vis >> (j + 1)) & 1u) ? y1 : 0.f;
        float g0, g1;
        fsub2(g0, g1, __uint_as_float(dv[j]), __uint_as_float(dv[j + 1]), Dq, Dq);
        fmul2(g0, g1, p0, p1, g0, g1);
        w[j2] = pack_bf16(g0, g1);
      }
      BTRACE(3, it);
      tmem_st16(tb + hf * 32, w);
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&ds_full[it & 1]);
      BTRACE(4, it);
    }
    __nv_bfloat16* out = a.dqkv + static_cast<size_t>(q) * a.ld_dqkv + a.q_col0 + h * HD + hf * 64;
    if (it > 0) {
      mbar_wait(dq_done, 0);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < 64; c += 32) {
        uint32_t o[32];
        tmem_ld32(tmem + lane_off + 256 + hf * 64 + c, o);
        tmem_ld_wait();
        if (row_ok) {
          uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 16; ++j)
            pk[j] = pack_bf16(__uint_as_float(o[2 * j]) * a.scale, __uint_as_float(o[2 * j + 1]) * a.scale);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            reinterpret_cast<uint4*>(out + c)[j] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
        }
      }
    } else if (row_ok) {
      for (int c = 0; c < 64; c += 8) *reinterpret_cast<uint4*>(out + c) = make_uint4(0, 0, 0, 0);
    }
  }
  BTRACE_FINISH;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// D[h][q] = sum_c dO[q][128 h + c] * O[q][128 h + c] (fp32), one warp per (q, h).
__global__ void attn_bwd_prep_kernel(const __nv_bfloat16* __restrict__ dO, int ldo,
                                     const __nv_bfloat16* __restrict__ O, int ld_o, int L,
                                     int n_heads, float* __restrict__ D, int ld_stat) {
  const long w = (static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= static_cast<long>(L) * n_heads) return;
  const int q = static_cast<int>(w / n_heads), h = static_cast<int>(w % n_heads);
  const uint2 g = *reinterpret_cast<const uint2*>(dO + static_cast<size_t>(q) * ldo + h * 128 + lane * 4);
  const uint2 o = *reinterpret_cast<const uint2*>(O + static_cast<size_t>(q) * ld_o + h * 128 + lane * 4);
  const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&g);
  const __nv_bfloat162* o2 = reinterpret_cast<const __nv_bfloat162*>(&o);
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float2 a = __bfloat1622float2(g2[i]), b = __bfloat1622float2(o2[i]);
    s = fmaf(a.x, b.x, s);
    s = fmaf(a.y, b.y, s);
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) D[static_cast<size_t>(h) * ld_stat + q] = s;
}

// ---------------------------------------------------------------------------
// Elementwise / reduction kernels of the backward pass (HBM-bound).
constexpr int NORM_ROWS = 64;  // rows per CTA (one dw partial per chunk)
constexpr int NORM_MAXC = 16;  // columns per thread: d <= 16 * 256

__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();  // red may still be read by a previous call
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
  for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) t += red[i];  // fixed order
  return t;
}

__global__ void __launch_bounds__(256) rmsnorm_bwd_kernel(
    const float* __restrict__ x, int ldx, const float* __restrict__ w, const float* __restrict__ dy,
    int ldy, float* __restrict__ dx, int ld_dx, int n, int d, float eps, const int* __restrict__ rows,
    float* __restrict__ dw_part) {
  __shared__ float red[8];
  float dwp[NORM_MAXC];
#pragma unroll
  for (int t = 0; t < NORM_MAXC; ++t) dwp[t] = 0.f;
  const int r0 = blockIdx.x * NORM_ROWS, r1 = min(n, r0 + NORM_ROWS);
  for (int i = r0; i < r1; ++i) {
    const long row = rows ? rows[i] : i;
    const float* xr = x + row * ldx;
    const float* gr = dy + static_cast<long>(i) * ldy;
    float ss = 0.f, dot = 0.f;
#pragma unroll
    for (int t = 0; t < NORM_MAXC; ++t) {
      const int j = threadIdx.x + 256 * t;
      if (j < d) {
        const float xv = xr[j];
        ss = fmaf(xv, xv, ss);
        dot = fmaf(w[j] * gr[j], xv, dot);
      }
    }
    ss = block_sum(ss, red);
    dot = block_sum(dot, red);
    const float r = rsqrtf(ss / static_cast<float>(d) + eps);
    const float c = r * r * r * dot / static_cast<float>(d);
    float* dr = dx + row * ld_dx;
#pragma unroll
    for (int t = 0; t < NORM_MAXC; ++t) {
      const int j = threadIdx.x + 256 * t;
      if (j < d) {
        const float xv = xr[j], g = gr[j];
        dr[j] += r * w[j] * g - xv * c;
        dwp[t] = fmaf(g * xv, r, dwp[t]);
      }
    }
  }
#pragma unroll
  for (int t = 0; t < NORM_MAXC; ++t) {
    const int j = threadIdx.x + 256 * t;
    if (j < d) dw_part[static_cast<size_t>(blockIdx.x) * d + j] = dwp[t];
  }
}

// out[c] += sum over chunks of part[chunk][c], chunks in order (deterministic;
// the gradients of a group are zeroed once and every SP rank adds its share)
__global__ void chunk_sum_kernel(const float* __restrict__ part, int n_chunks, int n_cols,
                                 float* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_cols) return;
  float s = 0.f;
  for (int k = 0; k < n_chunks; ++k) s += part[static_cast<size_t>(k) * n_cols + c];
  out[c] += s;
}

constexpr int COLSUM_ROWS = 128;
__global__ void colsum_part_kernel(const __nv_bfloat16* __restrict__ X, int ld, int n_rows,
                                   int n_cols, float* __restrict__ part) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_cols) return;
  const int r0 = blockIdx.y * COLSUM_ROWS, r1 = min(n_rows, r0 + COLSUM_ROWS);
  float s = 0.f;
  for (int r = r0; r < r1; ++r) s += __bfloat162float(X[static_cast<size_t>(r) * ld + c]);
  part[static_cast<size_t>(blockIdx.y) * n_cols + c] = s;
}

__global__ void cast_f32_bf16_kernel(const float* __restrict__ in, int ld_in,
                                     __nv_bfloat16* __restrict__ out, int ld_out, int n_rows,
                                     int n_cols) {
  const long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int pairs = n_cols / 2;
  if (i >= static_cast<long>(n_rows) * pairs) return;
  const long r = i / pairs;
  const int c = static_cast<int>(i % pairs) * 2;
  const float2 v = *reinterpret_cast<const float2*>(in + r * ld_in + c);
  *reinterpret_cast<__nv_bfloat162*>(out + r * ld_out + c) = __floats2bfloat162_rn(v.x, v.y);
}

__global__ void slot_sum_kernel(const float* __restrict__ slots, int n_slots, long stride, long n,
                                float* __restrict__ out) {
  const long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float v = slots[i];
  for (int q = 1; q < n_slots; ++q) v += slots[q * stride + i];
  out[i] = v;
}

__global__ void fill_f32_kernel(float* __restrict__ out, int n, float v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = v;
}

__global__ void negate_i32_kernel(const int* __restrict__ in, int* __restrict__ out, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = -in[i];
}

__global__ void embed_grad_kernel(const float* __restrict__ dh, int d, const int* __restrict__ seg_tok,
                                  const int* __restrict__ seg_off, const int* __restrict__ positions,
                                  float* __restrict__ dE) {
  const int sg = blockIdx.x;
  const int b = seg_off[sg], e = seg_off[sg + 1];
  float* out = dE + static_cast<size_t>(seg_tok[sg]) * d;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float s = 0.f;
    for (int i = b; i < e; ++i) s += dh[static_cast<size_t>(positions[i]) * d + c];
    out[c] += s;
  }
}

__global__ void grpo_coeff_kernel(const float* __restrict__ lp, const float* __restrict__ old_lp,
                                  const float* __restrict__ lp_ref, const float* __restrict__ adv,
                                  const int* __restrict__ lengths, int G, int n_tokens,
                                  double clip_eps, double beta, int sampled, float* __restrict__ coef) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= G) return;
  long off = 0;
  for (int i = 0; i < g; ++i) off += lengths[i];
  const double A = adv[g];
  const double tok_w = 1.0 / (static_cast<double>(G) * lengths[g]);
  const double kl_w = -beta / static_cast<double>(n_tokens);
  for (int t = 0; t < lengths[g]; ++t) {
    const double l = lp[off + t];
    const double ratio = exp(l - static_cast<double>(old_lp[off + t]));
    const bool plateau = (A > 0 && ratio > 1.0 + clip_eps) || (A < 0 && ratio < 1.0 - clip_eps);
    double c = (A != 0.0 && !plateau) ? tok_w * A * ratio : 0.0;
    if (sampled && beta != 0.0) c += kl_w * (1.0 - exp(static_cast<double>(lp_ref[off + t]) - l));
    coef[off + t] = static_cast<float>(c);
  }
}

// seq -> heads: one CTA per sequence row of this rank.
__global__ void route_seq_to_heads_kernel(RouteArgs ra, long b, const __nv_bfloat16* __restrict__ dO,
                                          int ld_do, const float* __restrict__ Dseq, int ld_dseq) {
  const int r = blockIdx.x;
  const long q = b + r;
  const int blk = static_cast<int>(q / ATTN_ROW_BLOCK);
  for (int p = 0; p < ra.K; ++p) {
    const RouteRank& P = ra.r[p];
    const int nqp = P.q_hi - P.q_lo;
    if (nqp <= 0) continue;
    if (P.rparts > 1 && attn_row_part(blk, ra.n_blocks, P.rparts) != P.rpart) continue;
    const uint4* src = reinterpret_cast<const uint4*>(dO + static_cast<size_t>(r) * ld_do + P.q_lo * 128);
    uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(P.doh) + q * nqp * 128);
    for (int i = threadIdx.x; i < nqp * 16; i += blockDim.x) dst[i] = src[i];
    for (int h = threadIdx.x; h < nqp; h += blockDim.x)
      P.Dh[static_cast<size_t>(h) * P.ld_stat + q] = Dseq[static_cast<size_t>(P.q_lo + h) * ld_dseq + r];
  }
}

// heads -> seq: one CTA per sequence row (all L rows) of head rank p.
__global__ void route_heads_to_seq_kernel(RouteArgs ra, int p, const __nv_bfloat16* __restrict__ dqkvh,
                                          int ld_h, const float* __restrict__ dkv32, int ld32) {
  const long q = blockIdx.x;
  const RouteRank& P = ra.r[p];
  int o = 0;
  while (o + 1 < ra.K && q >= ra.r[o + 1].b) ++o;
  const RouteRank& Ow = ra.r[o];
  const long row = q - Ow.b;
  const int nqp = P.q_hi - P.q_lo, nkvp = P.kv_hi - P.kv_lo;
  const int Cqkv = (ra.nq + 2 * ra.nkv) * 128;
  const int m = ra.K / ra.nkv > 1 ? ra.K / ra.nkv : 1;  // ranks sharing a kv head
  const uint4* src = reinterpret_cast<const uint4*>(dqkvh + q * ld_h);
  __nv_bfloat16* drow = static_cast<__nv_bfloat16*>(Ow.dqkv) + row * Cqkv;
  const bool own = P.rparts <= 1 ||
                   attn_row_part(static_cast<int>(q / ATTN_ROW_BLOCK), ra.n_blocks, P.rparts) == P.rpart;
  if (own) {  // dq of this rank's query heads
    uint4* dst = reinterpret_cast<uint4*>(drow + P.q_lo * 128);
    for (int i = threadIdx.x; i < nqp * 16; i += blockDim.x) dst[i] = src[i];
  }
  if (m == 1) {
    const uint4* sk = src + nqp * 16;
    const uint4* sv = src + (nqp + nkvp) * 16;
    uint4* dk = reinterpret_cast<uint4*>(drow + (ra.nq + P.kv_lo) * 128);
    uint4* dv = reinterpret_cast<uint4*>(drow + (ra.nq + ra.nkv + P.kv_lo) * 128);
    for (int i = threadIdx.x; i < nkvp * 16; i += blockDim.x) {
      dk[i] = sk[i];
      dv[i] = sv[i];
    }
  } else {  // fp32 partial: this rank's slot of the owner's [m][n][2 n_kv 128] buffer
    const float4* s32 = reinterpret_cast<const float4*>(dkv32 + q * ld32);
    float* srow = static_cast<float*>(Ow.slots) +
                  (static_cast<size_t>(P.slot) * (Ow.e - Ow.b) + row) * (2 * ra.nkv * 128);
    float4* dk = reinterpret_cast<float4*>(srow + P.kv_lo * 128);
    float4* dv = reinterpret_cast<float4*>(srow + (ra.nkv + P.kv_lo) * 128);
    for (int i = threadIdx.x; i < nkvp * 32; i += blockDim.x) {
      dk[i] = s32[i];
      dv[i] = s32[nkvp * 32 + i];
    }
  }
}

// dk | dv columns of dqkv = sum over the m slots in slot order (fp32, one
// rounding to bf16).
__global__ void kv_partial_sum_kernel(const float* __restrict__ slots, int m, long n, int nkv,
                                      __nv_bfloat16* __restrict__ dqkv, int nq) {
  const long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int w = 2 * nkv * 128;
  if (i >= n * w) return;
  const long row = i / w;
  const int c = static_cast<int>(i % w);
  float v = 0.f;
  for (int j = 0; j < m; ++j) v += slots[(static_cast<size_t>(j) * n + row) * w + c];
  const int Cqkv = (nq + 2 * nkv) * 128;
  dqkv[row * Cqkv + nq * 128 + c] = __float2bfloat16_rn(v);
}

}  // namespace

void attention_bwd(const AttnBwdParams& p, cudaStream_t stream) {
  MRSP_REQUIRE(p.L > 0 && p.n_heads > 0 && p.q_per_kv > 0 && p.n_heads % p.q_per_kv == 0,
               MRSP_INVALID_ARGUMENT, "attention_bwd: empty problem");
  MRSP_REQUIRE(p.row_parts >= 1 && p.row_part >= 0 && p.row_part < p.row_parts,
               MRSP_INVALID_ARGUMENT, "attention_bwd: bad query-row split");
  MRSP_REQUIRE(p.ld_qkv % 8 == 0 && p.ld_do % 8 == 0 && p.ld_o % 8 == 0 && p.ld_dqkv % 8 == 0 &&
                   p.ld_stat % 4 == 0 && p.ld_stat >= p.L,
               MRSP_INVALID_ARGUMENT, "attention_bwd: leading dims");
  MRSP_REQUIRE(p.Lmax > 0 || p.Lp >= p.L, MRSP_INVALID_ARGUMENT, "attention_bwd: bad mask");
  static const bool attr = [] {
    MRSP_CUDA(cudaFuncSetAttribute(attn_bwd_dq, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(DQ_SMEM)));
    MRSP_CUDA(cudaFuncSetAttribute(attn_bwd_dkdv, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(KV_SMEM)));
    MRSP_CUDA(cudaFuncSetAttribute(attn_bwd_dq2<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(DQ2_SMEM)));
    MRSP_CUDA(cudaFuncSetAttribute(attn_bwd_dq2<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(DQ2_SMEM)));
    MRSP_CUDA(cudaFuncSetAttribute(attn_bwd_dq2<true, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(DQ2_SMEM)));
    MRSP_CUDA(cudaFuncSetAttribute(attn_bwd_dq2<true, 12>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(DQ2_SMEM)));
    MRSP_CUDA(cudaFuncSetAttribute(attn_bwd_dkdv2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(KV2_SMEM)));
    MRSP_CUDA(cudaFuncSetAttribute(attn_bwd_dkdv4<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(V4_SMEM)));
    MRSP_CUDA(cudaFuncSetAttribute(attn_bwd_dkdv4<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(V4_SMEM)));
    MRSP_CUDA(cudaFuncSetAttribute(attn_bwd_dkdv4<12>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(V4_SMEM)));
    return true;
  }();
  // MRSP_ATTN_BWD=1: the single-buffered v1 kernels; =2: v2 (dQ with Q / dO
  // in shared memory, dK / dV in 64-query halves); =3: v2 with the TMEM-operand
  // dQ kernel; default 4: that dQ kernel and the v4 dK / dV kernel
  static const int version = [] {
    const char* v = std::getenv("MRSP_ATTN_BWD");
    return v ? std::atoi(v) : 4;
  }();
  (void)attr;
  // D = rowsum(dO o O) into the workspace p.D (unless the caller provides it)
  if (!p.d_given) {
    const long warps = static_cast<long>(p.L) * p.n_heads;
    attn_bwd_prep_kernel<<<static_cast<unsigned>((warps * 32 + 255) / 256), 256, 0, stream>>>(
        static_cast<const __nv_bfloat16*>(p.dO), p.ld_do, static_cast<const __nv_bfloat16*>(p.O),
        p.ld_o, p.L, p.n_heads, p.D, p.ld_stat);
    count_launch();
    MRSP_CUDA(cudaGetLastError());
  }
  BwdArgs a;
  a.L = p.L;
  a.Lp = p.Lp;
  a.Lmax = p.Lmax > 0 ? p.Lmax : 1;
  a.n_heads = p.n_heads;
  a.q_per_kv = p.q_per_kv;
  a.q_col0 = p.q_col0;
  a.k_col0 = p.k_col0;
  a.v_col0 = p.v_col0;
  a.scale = p.scale;
  a.scale_log2 = p.scale * 1.4426950408889634f;
  a.lse = p.lse;
  a.D = p.D;
  a.ld_stat = p.ld_stat;
  a.dqkv = static_cast<__nv_bfloat16*>(p.dqkv);
  a.ld_dqkv = p.ld_dqkv;
  a.row_parts = p.row_parts;
  a.row_part = p.row_part;
  a.dkv32 = p.dkv32;
  a.ld_dkv32 = p.ld_dkv32;
  a.qkv = static_cast<const __nv_bfloat16*>(p.qkv);
  a.ld_qkv = p.ld_qkv;
  a.dO = static_cast<const __nv_bfloat16*>(p.dO);
  a.ld_do = p.ld_do;
  a.n_blocks = (p.L + ATTN_ROW_BLOCK - 1) / ATTN_ROW_BLOCK;
  a.n_local_blocks = 0;
  if (p.row_parts > 1)
    while (attn_row_block(a.n_local_blocks, p.row_part, a.n_blocks, p.row_parts) >= 0) ++a.n_local_blocks;
  CUtensorMap tqkv = make_tmap_bf16_2d(p.qkv, p.L, p.ld_qkv, p.ld_qkv, 128, 64);
  CUtensorMap tdo = make_tmap_bf16_2d(p.dO, p.L, p.ld_do, p.ld_do, 128, 64);
  CUtensorMap tlse = make_tmap_f32_2d(p.lse, p.n_heads, p.L, p.ld_stat, 1, 128, CU_TENSOR_MAP_SWIZZLE_NONE);
  CUtensorMap td = make_tmap_f32_2d(p.D, p.n_heads, p.L, p.ld_stat, 1, 128, CU_TENSOR_MAP_SWIZZLE_NONE);
  const int n_qt = (p.L + TQ - 1) / TQ, n_kt = (p.L + TK - 1) / TK;
  const int n_tiles = p.row_parts > 1 ? 2 * a.n_local_blocks : n_qt;
  if (version == 1) {
    MRSP_REQUIRE(p.row_parts == 1 && p.dkv32 == nullptr, MRSP_INVALID_ARGUMENT,
                 "attention_bwd: the v1 kernels have no query-row split / fp32 partials");
    attn_bwd_dq<<<n_qt * p.n_heads, THREADS, DQ_SMEM, stream>>>(tqkv, tdo, a);
    count_launch();
    MRSP_CUDA(cudaGetLastError());
    attn_bwd_dkdv<<<n_kt * (p.n_heads / p.q_per_kv), THREADS, KV_SMEM, stream>>>(tqkv, tdo, tlse, td, a);
    count_launch();
    MRSP_CUDA(cudaGetLastError());
    return;
  }
  CUtensorMap t64 = make_tmap_bf16_2d(p.qkv, p.L, p.ld_qkv, p.ld_qkv, 64, 64);
  CUtensorMap tdo64 = make_tmap_bf16_2d(p.dO, p.L, p.ld_do, p.ld_do, 64, 64);
  CUtensorMap tlse64 = make_tmap_f32_2d(p.lse, p.n_heads, p.L, p.ld_stat, 1, 64, CU_TENSOR_MAP_SWIZZLE_NONE);
  CUtensorMap td64 = make_tmap_f32_2d(p.D, p.n_heads, p.L, p.ld_stat, 1, 64, CU_TENSOR_MAP_SWIZZLE_NONE);
  if (n_tiles > 0) {
    static const int dq_poly = [] {
      const char* v = std::getenv("MRSP_ATTN_BWD_DQ_POLY");
      return v ? std::atoi(v) : 0;
    }();
    if (version >= 3 && dq_poly >= 12)
      attn_bwd_dq2<true, 12><<<n_tiles * p.n_heads, THREADS, DQ2_SMEM, stream>>>(tqkv, t64, tdo, a);
    else if (version >= 3 && dq_poly >= 8)
      attn_bwd_dq2<true, 8><<<n_tiles * p.n_heads, THREADS, DQ2_SMEM, stream>>>(tqkv, t64, tdo, a);
    else if (version >= 3)
      attn_bwd_dq2<true><<<n_tiles * p.n_heads, THREADS, DQ2_SMEM, stream>>>(tqkv, t64, tdo, a);
    else
      attn_bwd_dq2<false><<<n_tiles * p.n_heads, THREADS, DQ2_SMEM, stream>>>(tqkv, t64, tdo, a);
    count_launch();
    MRSP_CUDA(cudaGetLastError());
  }
  // dK / dV v4: pairs (of 32) whose exp2 runs on the FMA pipe (8 measured 2%
  // faster at c3 than 0 or 12, profiles/r1_attention_study.md §7c)
  static const int bwd_poly = [] {
    const char* v = std::getenv("MRSP_ATTN_BWD_POLY");
    return v ? std::atoi(v) : 8;
  }();
  const int n_kv_ctas = n_kt * (p.n_heads / p.q_per_kv);
  if (version >= 4 && bwd_poly >= 12)
    attn_bwd_dkdv4<12><<<n_kv_ctas, THREADS, V4_SMEM, stream>>>(tqkv, tdo, tlse, td, a);
  else if (version >= 4 && bwd_poly >= 8)
    attn_bwd_dkdv4<8><<<n_kv_ctas, THREADS, V4_SMEM, stream>>>(tqkv, tdo, tlse, td, a);
  else if (version >= 4)
    attn_bwd_dkdv4<0><<<n_kv_ctas, THREADS, V4_SMEM, stream>>>(tqkv, tdo, tlse, td, a);
  else
    attn_bwd_dkdv2<<<n_kt * (p.n_heads / p.q_per_kv), THREADS, KV2_SMEM, stream>>>(tqkv, t64, tdo64, tlse64,
                                                                                    td64, a);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

}  // namespace mrsp

namespace mrsp {

size_t rmsnorm_bwd_workspace_bytes(int n, int d) {
  return static_cast<size_t>((n + NORM_ROWS - 1) / NORM_ROWS) * d * 4 + 256;
}

void rmsnorm_bwd(const float* x, int ldx, const float* w, const float* dy, int ldy, float* dx_acc,
                 int ld_dx, int n, int d, float eps, const int* rows, float* dw_out, void* ws,
                 cudaStream_t s) {
  if (n <= 0) return;
  MRSP_REQUIRE(d <= NORM_MAXC * 256, MRSP_INVALID_ARGUMENT, "rmsnorm_bwd: d too large");
  const int chunks = (n + NORM_ROWS - 1) / NORM_ROWS;
  float* part = static_cast<float*>(ws);
  rmsnorm_bwd_kernel<<<chunks, 256, 0, s>>>(x, ldx, w, dy, ldy, dx_acc, ld_dx, n, d, eps, rows, part);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
  if (dw_out) {
    chunk_sum_kernel<<<(d + 255) / 256, 256, 0, s>>>(part, chunks, d, dw_out);
    count_launch();
    MRSP_CUDA(cudaGetLastError());
  }
}

size_t colsum_workspace_bytes(int n_rows, int n_cols) {
  return static_cast<size_t>((n_rows + COLSUM_ROWS - 1) / COLSUM_ROWS) * n_cols * 4 + 256;
}

void colsum_bf16(const __nv_bfloat16* X, int ld, int n_rows, int n_cols, float* out, void* ws,
                 cudaStream_t s) {
  if (n_rows <= 0) return;
  const int chunks = (n_rows + COLSUM_ROWS - 1) / COLSUM_ROWS;
  float* part = static_cast<float*>(ws);
  colsum_part_kernel<<<dim3((n_cols + 255) / 256, chunks), 256, 0, s>>>(X, ld, n_rows, n_cols, part);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
  chunk_sum_kernel<<<(n_cols + 255) / 256, 256, 0, s>>>(part, chunks, n_cols, out);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

void cast_f32_bf16(const float* in, int ld_in, __nv_bfloat16* out, int ld_out, int n_rows,
                   int n_cols, cudaStream_t s) {
  MRSP_REQUIRE(n_cols % 2 == 0 && ld_in % 2 == 0 && ld_out % 2 == 0, MRSP_INVALID_ARGUMENT,
               "cast_f32_bf16: even widths");
  const long n = static_cast<long>(n_rows) * (n_cols / 2);
  if (n == 0) return;
  cast_f32_bf16_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(in, ld_in, out, ld_out,
                                                                             n_rows, n_cols);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

void slot_sum_f32(const float* slots, int n_slots, long slot_stride, long n, float* out,
                  cudaStream_t s) {
  if (n <= 0) return;
  slot_sum_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(slots, n_slots, slot_stride, n, out);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

void fill_f32(float* out, int n, float v, cudaStream_t s) {
  if (n <= 0) return;
  fill_f32_kernel<<<(n + 255) / 256, 256, 0, s>>>(out, n, v);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

void negate_i32(const int* in, int* out, int n, cudaStream_t s) {
  if (n <= 0) return;
  negate_i32_kernel<<<(n + 255) / 256, 256, 0, s>>>(in, out, n);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

void embed_grad(const float* dh, int d, const int* seg_tok, const int* seg_off,
                const int* positions, int n_seg, float* dE, cudaStream_t s) {
  if (n_seg <= 0) return;
  embed_grad_kernel<<<n_seg, 256, 0, s>>>(dh, d, seg_tok, seg_off, positions, dE);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

void grpo_token_coeffs(const float* lp, const float* old_lp, const float* lp_ref,
                       const float* adv, const int* lengths, int G, int n_tokens, double clip_eps,
                       double kl_beta, int sampled_kl, float* coef, cudaStream_t s) {
  if (G <= 0 || n_tokens <= 0) return;
  grpo_coeff_kernel<<<(G + 127) / 128, 128, 0, s>>>(lp, old_lp, lp_ref, adv, lengths, G, n_tokens,
                                                    clip_eps, kl_beta, sampled_kl, coef);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

}  // namespace mrsp

using namespace mrsp;

extern "C" mrsp_status mrsp_op_attention_lse(const void* Q, int ldq, int q_col0, const void* K,
                                             int ldk, int k_col0, const void* V, int ldv,
                                             int v_col0, void* O, int ldo, int o_col0, int L,
                                             int n_heads, int q_per_kv, float scale, int Lp,
                                             int Lmax, float* lse, int lse_ld, void* stream) {
  return guard([&] {
    require_device();
    AttnParams p{Q, ldq, q_col0, K, ldk, k_col0, V, ldv, v_col0, O, ldo, o_col0,
                 L, n_heads, q_per_kv, scale, ATTN_CAUSAL_PREFIX, Lp, Lmax, 0};
    p.lse = lse;
    p.lse_ld = lse_ld;
    attention_fwd(p, static_cast<cudaStream_t>(stream));
  });
}

extern "C" mrsp_status mrsp_op_attention_bwd(const void* qkv, int ld_qkv, int q_col0, int k_col0,
                                             int v_col0, const void* O, int ld_o, const void* dO,
                                             int ld_do, const float* lse, float* D, int ld_stat,
                                             void* dqkv, int ld_dqkv, int L, int n_heads,
                                             int q_per_kv, float scale, int Lp, int Lmax,
                                             void* stream) {
  return guard([&] {
    require_device();
    AttnBwdParams p{qkv, ld_qkv, q_col0, k_col0, v_col0, O, ld_o, dO, ld_do, lse, D, ld_stat,
                    dqkv, ld_dqkv, L, n_heads, q_per_kv, scale, Lp, Lmax};
    attention_bwd(p, static_cast<cudaStream_t>(stream));
  });
}

extern "C" mrsp_status mrsp_op_rmsnorm_bwd(const float* x, int ldx, const float* w,
                                           const float* dy, int ldy, float* dx_acc, int ld_dx,
                                           int n, int d, float eps, const int32_t* rows,
                                           float* dw_out, void* stream) {
  return guard([&] {
    require_device();
    void* ws = nullptr;
    const size_t b = rmsnorm_bwd_workspace_bytes(n, d);
    MRSP_CUDA(cudaMallocAsync(&ws, b, static_cast<cudaStream_t>(stream)));
    rmsnorm_bwd(x, ldx, w, dy, ldy, dx_acc, ld_dx, n, d, eps, rows, dw_out, ws,
                static_cast<cudaStream_t>(stream));
    MRSP_CUDA(cudaFreeAsync(ws, static_cast<cudaStream_t>(stream)));
  });
}

extern "C" mrsp_status mrsp_op_gemm_swiglu_bwd(const void* X, const void* W_gu, const void* dA,
                                               void* dGU, void* act, int M, int N, int K,
                                               void* stream) {
  return guard([&] {
    require_device();
    GemmArgs g{X, W_gu, dGU, M, N, K, K, K, N, GEMM_EPI_SWIGLU_BWD, nullptr, nullptr, 0};
    g.aux = dA;
    g.ld_aux = N / 2;
    g.aux_out = act;
    g.ld_aux_out = N / 2;
    gemm_bf16(g, static_cast<cudaStream_t>(stream));
  });
}

extern "C" mrsp_status mrsp_op_lmhead_dual_dlogits(const void* X_policy, const void* W_policy,
                                                   const void* X_ref, const void* W_ref, int M,
                                                   int V, int K, const int32_t* targets,
                                                   const float* coef, float kw, const float* kl,
                                                   const float* lse_policy, const float* lse_ref,
                                                   void* G, int ldg, void* stream) {
  return guard([&] {
    require_device();
    lmhead_dual_dlogits(X_policy, W_policy, X_ref, W_ref, M, V, K, targets, coef, kw, kl,
                        lse_policy, lse_ref, G, ldg, static_cast<cudaStream_t>(stream));
  });
}

namespace mrsp {

void attention_rowdot(const void* dO, int ld_do, const void* O, int ld_o, int n, int n_heads,
                      float* D, int ld_d, cudaStream_t stream) {
  if (n <= 0 || n_heads <= 0) return;
  const long warps = static_cast<long>(n) * n_heads;
  attn_bwd_prep_kernel<<<static_cast<unsigned>((warps * 32 + 255) / 256), 256, 0, stream>>>(
      static_cast<const __nv_bfloat16*>(dO), ld_do, static_cast<const __nv_bfloat16*>(O), ld_o, n,
      n_heads, D, ld_d);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

void route_seq_to_heads(const RouteArgs& ra, long b, long e, const void* dO, int ld_do,
                        const float* Dseq, int ld_dseq, cudaStream_t s) {
  if (e <= b) return;
  route_seq_to_heads_kernel<<<static_cast<unsigned>(e - b), 128, 0, s>>>(
      ra, b, static_cast<const __nv_bfloat16*>(dO), ld_do, Dseq, ld_dseq);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

void route_heads_to_seq(const RouteArgs& ra, int p, const void* dqkvh, int ld_h, const float* dkv32,
                        int ld32, cudaStream_t s) {
  if (ra.L <= 0) return;
  route_heads_to_seq_kernel<<<static_cast<unsigned>(ra.L), 128, 0, s>>>(
      ra, p, static_cast<const __nv_bfloat16*>(dqkvh), ld_h, dkv32, ld32);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

void kv_partial_sum(const void* slots, int m, long n, int nkv, void* dqkv, int nq, cudaStream_t s) {
  const long total = n * 2 * nkv * 128;
  if (total <= 0) return;
  kv_partial_sum_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, s>>>(
      static_cast<const float*>(slots), m, n, nkv, static_cast<__nv_bfloat16*>(dqkv), nq);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

}  // namespace mrsp
