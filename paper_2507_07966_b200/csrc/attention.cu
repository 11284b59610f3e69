// attention.cu — tcgen05 flash-attention forward for sm_100a (head dim 128).
//
// One CTA = TWO 128-query tiles of one query head, sharing every K/V tile.
// The tensor core (one elected thread of warp 1) alternates between the tiles:
//     ... P.V(t0, j-1) | S(t0, j) = Q0.K_j^T | P.V(t1, j-1) | S(t1, j) ...
// so while softmax warpgroup 0 turns S(t0) into P(t0) the tensor core works on
// tile 1 and vice versa (ping-pong). S and O accumulate in TMEM
// (S0 | S1 | O0 | O1 = 512 columns); K and V stream through a 5-slot TMA ring
// (K_j, V_j alternate). P never touches shared memory: the softmax writes it
// as packed bf16 over the first 64 columns of its S buffer (tcgen05.st) and
// the P.V MMA takes its A operand straight from TMEM.
//
// Softmax (thread = query row): tcgen05.ld of the 128 scores, row max on the
// raw scores (8 independent chains), p = exp2(s*scale - m) with packed
// FFMA2 / FADD2 (fp32x2) arithmetic and MUFU.EX2 (a packed degree-3 FMA-pipe
// exp2 is available as kPoly but measured no faster here); O is rescaled in TMEM only when the
// running max grows by > 2^8 (lazy rescale, warp-uniform because tcgen05.ld/st
// are warp-collective). Registers rebalanced with setmaxnreg (TMA/MMA
// warpgroup 56, softmax warpgroups 200).
//
// Roles (384 threads): warp 0 TMA, warp 1 MMA issuer, warp 2 TMEM allocator,
// warps 4-7 softmax of tile 0, warps 8-11 softmax of tile 1.
//
// Masks (MR-SP packed sequence):
//   ATTN_CAUSAL_PREFIX: sequence = [prefix (Lp) | G rows of Lmax]; query q sees
//     key k iff k <= q and (k < Lp or row(k) == row(q)) — every rollout row
//     attends to the shared prompt prefix and causally to itself only.
//   ATTN_BLOCK_DIAG: bidirectional inside blocks of `blk` tokens (one video
//     frame of the vision tower), nothing across blocks.
// Per (query tile, KV tile): skipped (no visible pair: no MMA, no softmax),
// full (no element mask) or partial (element mask).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "attention.h"
#include "common.h"
#include "sm100.cuh"
#include "tma.h"
#include "attn_common.cuh"

namespace mrsp {
namespace {

using namespace sm100;
using namespace attn_detail;

static_assert(2 * TQ == ATTN_ROW_BLOCK, "a CTA's query block is the row-split unit");
constexpr int CHUNK = 128 * 64 * 2;  // one 128-row x 64-col bf16 SW128 block (16 KB)
constexpr int TILE = 2 * CHUNK;      // a 128 x 128 bf16 operand (32 KB)
constexpr int RING = 5;              // K/V ring slots
constexpr int OFF_Q = 0;                       // Q0, Q1
constexpr int OFF_RING = OFF_Q + 2 * TILE;     // 5 slots
constexpr int OFF_BAR = OFF_RING + RING * TILE;
constexpr size_t SMEM_BYTES = 1024 + OFF_BAR + 256;
constexpr int THREADS = 384;
constexpr uint32_t TMEM_COLS = 512;  // S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512)
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 domain

// KV tile range covering both query tiles [q0, q0 + 256).
__device__ __forceinline__ void kt_range(int q0, const MaskDev& m, int n_kt, int& lo, int& hi) {
  const int qlast = q0 + 2 * TQ - 1;
  if (m.mode == ATTN_BLOCK_DIAG) {
    lo = (q0 / m.blk) * m.blk / TK;
    hi = min(n_kt, ((qlast / m.blk + 1) * m.blk + TK - 1) / TK);
  } else {
    lo = 0;
    hi = min(n_kt, qlast / TK + 1);
  }
}

// Next KV tile in [kt, hi) visible to either query tile; returns the two
// classes packed as c0 | c1 << 2 (0 when exhausted).
__device__ __forceinline__ int next_tile(int q0, int& kt, int hi, const MaskDev& m) {
  for (; kt < hi; ++kt) {
    const int c0 = tile_class(q0, kt, m), c1 = tile_class(q0 + TQ, kt, m);
    if (c0 | c1) return c0 | (c1 << 2);
  }
  return 0;
}

struct AttnArgs {
  int n_pairs, n_heads, q_per_kv;
  int n_local, row_parts, row_part;  // query blocks of this row part (all when 1 part)
  int q_col0, k_col0, v_col0, o_col0;
  // head stride in columns: HD (2-D maps, col0s in columns) or, when < HD,
  // the real head dim (3-D maps [rows][heads][hs], col0s in heads; the boxes'
  // columns past hs are zero-filled by TMA, so the tiles are hd-128 tiles)
  int hs;
  __nv_bfloat16* O;
  int ldo;
  float scale_log2;
  MaskDev mask;
  int n_dst, dst_ld, dst_col0;  // fused O scatter (AttnParams)
  long dst_bounds[9];
  __nv_bfloat16* dst_base[8];
  float* lse;  // optional [heads][lse_ld] (scaled log2 domain)
  int lse_ld;
};

// Destination row of query row q, head h: O itself, or the owner shard's buffer.
__device__ __forceinline__ __nv_bfloat16* out_row(const AttnArgs& a, int q, int h) {
  if (a.n_dst == 0) return a.O + static_cast<size_t>(q) * a.ldo + a.o_col0 + h * a.hs;
  int p = 0;
  while (p + 1 < a.n_dst && q >= a.dst_bounds[p + 1]) ++p;
  return a.dst_base[p] + static_cast<size_t>(q - a.dst_bounds[p]) * a.dst_ld + a.dst_col0 + h * a.hs;
}

// Work order: KV-head-major, then query-row blocks heaviest (longest KV sweep)
// first, then the q_per_kv query heads sharing that KV head. Every CTA of a
// wave then streams the same KV head's K/V (71 MB at c4 for K+V, fits the
// 126 MB L2) instead of all four heads' 285 MB — measured 44 GB of DRAM reads
// per c4 launch with head-minor order.
// With a query-row split the rank's share of blocks (attn_row_block) is walked
// in the same heaviest-first order.
__device__ __forceinline__ void work_item(int idx, const AttnArgs& a, int& block, int& h) {
  const int per_kv = a.n_local * a.q_per_kv;
  const int kvh = idx / per_kv;
  const int rem = idx - kvh * per_kv;
  const int li = rem / a.q_per_kv;
  block = a.row_parts > 1 ? attn_row_block(li, a.row_part, a.n_pairs, a.row_parts)
                          : a.n_pairs - 1 - li;
  h = kvh * a.q_per_kv + rem % a.q_per_kv;
}

// Optional per-phase timeline of one CTA (tools/ubench/attn_trace.cu builds
// this file with MRSP_ATTN_TRACE): lane 0 of a warp stamps clock() per event.
#ifdef MRSP_ATTN_TRACE
constexpr int kTraceCap = 8192;
#ifdef MRSP_ATTN_TRACE_GLOBAL
__device__ __forceinline__ uint32_t trace_clock() {  // ns, comparable across SMs
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return static_cast<uint32_t>(t);
}
#else
__device__ __forceinline__ uint32_t trace_clock() { return static_cast<uint32_t>(clock()); }
#endif
__device__ uint64_t g_attn_trace[24][kTraceCap];
__device__ int g_attn_trace_n[24];
__device__ int g_attn_trace_cta;
// traced: CTA g_attn_trace_cta, plus its cluster peer with the global clock
#ifdef MRSP_ATTN_TRACE_GLOBAL
#define ATRACE_ON ((blockIdx.x >> 1) == (g_attn_trace_cta >> 1))
#define ATRACE_ROW ((threadIdx.x >> 5) + 12 * (blockIdx.x & 1))
#else
#define ATRACE_ON (blockIdx.x == g_attn_trace_cta)
#define ATRACE_ROW (threadIdx.x >> 5)
#endif
#define ATRACE(ev, it)                                                                        \
  do {                                                                                        \
    if (ATRACE_ON && (threadIdx.x & 31) == 0 && trace_n < kTraceCap) {                        \
      g_attn_trace[ATRACE_ROW][trace_n++] =                                                   \
          (static_cast<uint64_t>(ev) << 56) | (static_cast<uint64_t>((it) & 0xffffff) << 32) | \
          static_cast<uint32_t>(trace_clock());                                               \
    }                                                                                         \
  } while (0)
#define ATRACE_INIT int trace_n = 0
#define ATRACE_FINISH \
  if (ATRACE_ON && (threadIdx.x & 31) == 0) g_attn_trace_n[ATRACE_ROW] = trace_n
#else
#define ATRACE(ev, it) \
  do {                 \
  } while (0)
#define ATRACE_INIT
#define ATRACE_FINISH
#endif

// kPoly: pairs (of every 32) whose exp2 runs on the FMA pipe (0 = all MUFU).
// kPC: chunks P is handed to the P.V MMA in (2: 64-key halves; 4: 32-key
// quarters, so the last chunk's MMA is shorter on the S -> P -> P.V chain).
// kSpec: the first chunk's exponentials are computed with the running max
// while the tile max is formed (redone on the rare max growth).
template <int kPoly, int kPC, int kSpec>
__global__ void __launch_bounds__(THREADS, 1)
    attn_fwd_tcgen05(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, AttnArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* r_full = bars + 1;    // [RING]
  uint64_t* r_empty = bars + 6;   // [RING]
  uint64_t* s_full = bars + 11;   // [2] per query tile
  uint64_t* s_free = bars + 13;   // [2]
  uint64_t* p_full = bars + 15;   // [2][4]: per query tile, per chunk of P
  uint64_t* pv_done = bars + 23;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 25);

  ATRACE_INIT;
  const int warp = warp_id();
  int pair, h;
  work_item(static_cast<int>(blockIdx.x), a, pair, h);
  const int kvh = h / a.q_per_kv;
  const int q0 = pair * 2 * TQ;
  const int n_kt = (a.mask.L + TK - 1) / TK;
  int kt_lo, kt_hi;
  kt_range(q0, a.mask, n_kt, kt_lo, kt_hi);

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    mbar_init(q_full, 1);
    for (int s = 0; s < RING; ++s) {
      mbar_init(&r_full[s], 1);
      mbar_init(&r_empty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&s_full[t], 1);
      mbar_init(&s_free[t], 128);
      for (int c = 0; c < 4; ++c) mbar_init(&p_full[4 * t + c], 128);
      mbar_init(&pv_done[t], 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    reg_dealloc<56>();
    if (warp == 0) {
      if (elect_one()) {
        // Q0, Q1 (rows past L are zero-filled by TMA)
        mbar_arrive_expect_tx(q_full, 2 * TILE);
        for (int t = 0; t < 2; ++t)
          for (int c = 0; c < 2; ++c) {
            if (a.hs == HD)
              tma_load_2d(smem + OFF_Q + t * TILE + c * CHUNK, &tmQ, q_full,
                          a.q_col0 + h * HD + c * 64, q0 + t * TQ);
            else
              tma_load_3d(smem + OFF_Q + t * TILE + c * CHUNK, &tmQ, q_full, c * 64,
                          a.q_col0 + h, q0 + t * TQ);
          }
        int slot = 0;
        uint32_t ph = 0;
        for (int kt = kt_lo; next_tile(q0, kt, kt_hi, a.mask); ++kt) {
          const int k0 = kt * TK;
          for (int kv = 0; kv < 2; ++kv) {  // K_j then V_j
            mbar_wait(&r_empty[slot], ph ^ 1);
            mbar_arrive_expect_tx(&r_full[slot], TILE);
            uint8_t* dst = smem + OFF_RING + slot * TILE;
            const CUtensorMap* tm = kv ? &tmV : &tmK;
            if (a.hs == HD) {
              const int col = (kv ? a.v_col0 : a.k_col0) + kvh * HD;
              tma_load_2d(dst, tm, &r_full[slot], col, k0);
              tma_load_2d(dst + CHUNK, tm, &r_full[slot], col + 64, k0);
            } else {
              const int head = (kv ? a.v_col0 : a.k_col0) + kvh;
              tma_load_3d(dst, tm, &r_full[slot], 0, head, k0);
              tma_load_3d(dst + CHUNK, tm, &r_full[slot], 64, head, k0);
            }
            if (++slot == RING) { slot = 0; ph ^= 1; }
          }
        }
      }
    } else if (warp == 1) {
      const uint32_t idesc_s = idesc_bf16_f32(TQ, TK);
      const uint32_t idesc_o = idesc_bf16_f32_bmn(TQ, HD);
      const uint32_t q_addr = smem_u32(smem + OFF_Q);
      const uint32_t ring_addr = smem_u32(smem + OFF_RING);
      mbar_wait(q_full, 0);
      int slot = 0;
      uint32_t ph = 0;
      int n_s[2] = {0, 0}, n_pv[2] = {0, 0};  // MMAs issued per query tile
      int pend_slot = -1;                     // ring slot of V_{j-1} (pending P.V)
      int pend_cls = 0;
      auto issue_s = [&](int t, uint32_t k_addr) {
        mbar_wait(&s_free[t], (n_s[t] & 1) ^ 1);
        ATRACE(10 + t, n_s[t]);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const uint32_t off = (kk / 4) * CHUNK + (kk % 4) * 32;
            mma_bf16_ss(tmem + t * 128, sdesc_sw128(q_addr + t * TILE + off),
                        sdesc_sw128(k_addr + off), idesc_s, kk > 0 ? 1u : 0u);
          }
          mma_commit(&s_full[t]);
        }
        __syncwarp();
        ATRACE(12 + t, n_s[t]);
        ++n_s[t];
      };
      auto issue_pv = [&](int t, uint32_t v_addr) {
        // kPC chunks of keys: the first chunks' MMAs start while the softmax
        // is still exponentiating the later ones
#pragma unroll
        for (int half = 0; half < kPC; ++half) {
          mbar_wait(&p_full[4 * t + half], n_pv[t] & 1);
          ATRACE(14 + 2 * t + (half * 2) / kPC, n_pv[t]);
          tc_fence_after();
          if (elect_one()) {
#pragma unroll
            for (int k4 = 0; k4 < 8 / kPC; ++k4) {
              const int kk = half * (8 / kPC) + k4;
              // A = P from TMEM (packed bf16 pairs over S(t)'s first 64 columns)
              const uint64_t bd = sdesc_sw128_mn(v_addr + kk * 2048, CHUNK);
              mma_bf16_ts(tmem + 256 + t * 128, tmem + t * 128 + kk * 8, bd, idesc_o,
                          (n_pv[t] > 0 || kk > 0) ? 1u : 0u);
            }
            if (half == kPC - 1) mma_commit(&pv_done[t]);
          }
          __syncwarp();
        }
        ++n_pv[t];
      };
      auto release = [&](int s) {
        if (elect_one()) mma_commit(&r_empty[s]);
        __syncwarp();
      };
      for (int kt = kt_lo;; ++kt) {
        const int cls = next_tile(q0, kt, kt_hi, a.mask);
        int k_slot = -1;
        if (cls) {  // K_j
          mbar_wait(&r_full[slot], ph);
          ATRACE(18, kt);
          k_slot = slot;
          if (++slot == RING) { slot = 0; ph ^= 1; }
        }
        const uint32_t k_addr = ring_addr + (k_slot < 0 ? 0 : k_slot) * TILE;
        const uint32_t v_addr = ring_addr + (pend_slot < 0 ? 0 : pend_slot) * TILE;
        // P.V(t0, j-1), S(t0, j), P.V(t1, j-1), S(t1, j)
        if (pend_slot >= 0 && (pend_cls & 3)) issue_pv(0, v_addr);
        if (cls & 3) issue_s(0, k_addr);
        if (pend_slot >= 0 && (pend_cls >> 2)) issue_pv(1, v_addr);
        if (cls >> 2) issue_s(1, k_addr);
        if (pend_slot >= 0) release(pend_slot);  // V_{j-1}: both P.V issued
        if (k_slot >= 0) release(k_slot);        // K_j: both S issued
        if (!cls) break;
        mbar_wait(&r_full[slot], ph);  // V_j becomes the pending P.V operand
        pend_slot = slot;
        pend_cls = cls;
        if (++slot == RING) { slot = 0; ph ^= 1; }
      }
    }
  } else {
    reg_alloc<200>();
    const int t = (warp - 4) >> 2;      // query tile of this warpgroup
    const int ew = (warp - 4) & 3;      // TMEM lane quarter
    const int r = ew * 32 + lane_id();  // query row in the tile
    const int q = q0 + t * TQ + r;
    const uint32_t lane_off = static_cast<uint32_t>(ew * 32) << 16;
    const uint32_t tS = tmem + t * 128 + lane_off;
    const uint32_t tO = tmem + 256 + t * 128 + lane_off;
    const float sl2 = a.scale_log2;
    // this row's visible key set, computed once: k < k_end and
    // (k < k_mid or k >= k_lo)   [k_mid = Lp, k_lo = start of the row's segment]
    int k_end, k_mid, k_lo;
    if (a.mask.mode == ATTN_BLOCK_DIAG) {
      k_lo = (q / a.mask.blk) * a.mask.blk;
      k_mid = 0;
      k_end = min(k_lo + a.mask.blk, a.mask.L);
    } else {
      k_end = min(q + 1, a.mask.L);
      k_mid = a.mask.Lp;
      k_lo = q >= a.mask.Lp ? a.mask.Lp + seg_of(q, a.mask) * a.mask.Lmax : 0;
    }
    float m_run = -INFINITY, l_run = 0.f;  // m_run in scaled log2 units
    int it = 0;                            // KV tiles processed by this warpgroup
    for (int kt = kt_lo;; ++kt) {
      const int both = next_tile(q0, kt, kt_hi, a.mask);
      if (!both) break;
      const int cls = (both >> (2 * t)) & 3;
      if (!cls) continue;
      mbar_wait(&s_full[t], it & 1);
      ATRACE(1, it);
      tc_fence_after();
      float s[TK];
      {
        uint32_t r0[32], r1[32], r2[32], r3[32];
        tmem_ld32(tS + 0, r0);
        tmem_ld32(tS + 32, r1);
        tmem_ld32(tS + 64, r2);
        tmem_ld32(tS + 96, r3);
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
      mbar_arrive(&s_free[t]);
      ATRACE(2, it);
      const int k0 = kt * TK;
      if (cls == 2) {
        // visible = k < k_end && (k < k_mid || k >= k_lo), as one bitmask per
        // 32 keys (2 instructions per element instead of ~5 of compares)
#pragma unroll
        for (int q = 0; q < TK / 32; ++q) {
          const int base = k0 + 32 * q;
          const uint32_t vis =
              lt_bits(k_end, base) & (lt_bits(k_mid, base) | ~lt_bits(k_lo, base));
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (!((vis >> j) & 1u)) s[32 * q + j] = -INFINITY;
        }
      }
      // 8 independent max chains (FMNMX3) instead of one 128-deep chain
      auto tile_max = [&]() {
        float m8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) m8[i] = fmaxf(s[i], s[i + 8]);
#pragma unroll
        for (int j = 16; j < TK; j += 16)
#pragma unroll
          for (int i = 0; i < 8; ++i) m8[i] = fmaxf(m8[i], fmaxf(s[j + i], s[j + i + 8]));
        return fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                     fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
      };
      constexpr int kPairs = 64 / kPC;  // packed bf16 pairs (TMEM columns) per chunk
      // p = 2^(s scale log2e - m) for chunk c of the tile, packed, row sums in acc
      auto exp_chunk = [&](int c, float neg_m, uint32_t (&w)[kPairs], float (&acc)[8]) {
#pragma unroll
        for (int i = 0; i < kPairs; ++i) {
          const int j = c * 2 * kPairs + 2 * i;
          float x0, x1;
          ffma2(x0, x1, s[j], s[j + 1], sl2, sl2, neg_m, neg_m);
          float p0, p1;
          if (poly_pair<kPoly>((c * kPairs + i) & 31)) {
            exp2_poly2(x0, x1, p0, p1);
          } else {
            p0 = exp2_mufu(x0);
            p1 = exp2_mufu(x1);
          }
          fadd2(acc[2 * (i & 3)], acc[2 * (i & 3) + 1], p0, p1);
          w[i] = pack_bf16(p0, p1);
        }
      };
      // the lazy rescale: the running max moves only when the tile's max
      // exceeds it by > 2^8; O and l are rescaled once the previous P.V is done
      auto rescale = [&](float mt, bool need) {
        if (it > 0) mbar_wait(&pv_done[t], (it - 1) & 1);
        tc_fence_after();
        if (__any_sync(0xffffffffu, need) && it > 0) {
          const float alpha = (need && m_run != -INFINITY) ? exp2f(m_run - mt) : 1.0f;
          if (need) l_run *= alpha;
#pragma unroll 1
          for (int c = 0; c < HD; c += 32) {
            uint32_t o[32];
            tmem_ld32(tO + c, o);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * alpha);
            tmem_st32(tO + c, o);
          }
          tmem_st_wait();
        }
        if (need) m_run = mt;
      };
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // 4 packed partial sums
      uint32_t w0[kPairs];
      float neg_m;
      if (kSpec && it > 0) {
        // Speculative: chunk 0's exponentials with the running max while the
        // tile max is formed alongside (MUFU and ALU pipes), so the max is off
        // the S -> P chain. Only when the max grows by > 2^8 (rare after the
        // first tiles) is chunk 0 redone after the rescale — the same results
        // as max-first, bit for bit.
        neg_m = m_run == -INFINITY ? 0.f : -m_run;
        exp_chunk(0, neg_m, w0, acc);
        const float mt = tile_max() * sl2;  // -inf stays -inf
        const bool need = mt > m_run + RESCALE_THRESHOLD;
        ATRACE(3, it);
        if (__any_sync(0xffffffffu, need)) {
          rescale(mt, need);
          neg_m = m_run == -INFINITY ? 0.f : -m_run;
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[i] = 0.f;
          exp_chunk(0, neg_m, w0, acc);
        }
      } else {
        const float mt = tile_max() * sl2;
        ATRACE(3, it);
        rescale(mt, mt > m_run + RESCALE_THRESHOLD);
        neg_m = m_run == -INFINITY ? 0.f : -m_run;
        exp_chunk(0, neg_m, w0, acc);
      }
#pragma unroll
      for (int c = 0; c < kPC; ++c) {
        uint32_t wc[kPairs];
        if (c > 0) exp_chunk(c, neg_m, wc, acc);
        const uint32_t (&w)[kPairs] = c == 0 ? w0 : wc;
        ATRACE(6 + (c * 2) / kPC, it);
        if constexpr (kPairs == 32) {
          tmem_st32(tS + c * 32, w);
        } else {
          tmem_st16(tS + c * 16, w);
        }
        tmem_st_wait();
        ATRACE(8 + (c * 2) / kPC, it);
        tc_fence_before();
        mbar_arrive(&p_full[4 * t + c]);  // this chunk of P is ready for the MMA
        ATRACE(4 + (c * 2) / kPC, it);
      }
      l_run += ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
      ++it;
    }
    // epilogue: O / l -> bf16 global
    const bool row_ok = q < a.mask.L;
    __nv_bfloat16* orow = row_ok ? out_row(a, q, h) : nullptr;
    if (a.lse != nullptr && row_ok)
      a.lse[static_cast<size_t>(h) * a.lse_ld + q] = l_run > 0.f ? m_run + log2f(l_run) : INFINITY;
    if (it > 0) {
      mbar_wait(&pv_done[t], (it - 1) & 1);
      tc_fence_after();
      const float inv_l = l_run > 0.f ? 1.0f / l_run : 0.f;
#pragma unroll 1
      for (int c = 0; c < a.hs; c += 32) {  // the head's hs columns (O past hs is 0)
        uint32_t o[32];
        tmem_ld32(tO + c, o);
        tmem_ld_wait();
        if (row_ok) {
          uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 16; ++j)
            pk[j] = pack_bf16(__uint_as_float(o[2 * j]) * inv_l, __uint_as_float(o[2 * j + 1]) * inv_l);
          uint4* dst = reinterpret_cast<uint4*>(orow + c);
          const int nv = min(4, (a.hs - c) / 8);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (j < nv) dst[j] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
        }
      }
    } else if (row_ok) {  // no visible key (only possible for rows past L)
      for (int c = 0; c < a.hs; c += 8) *reinterpret_cast<uint4*>(orow + c) = make_uint4(0, 0, 0, 0);
    }
  }
  ATRACE_FINISH;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<TMEM_COLS>(tmem);
}

// FMA-pipe exp2 share: measured no gain at c4 with P in TMEM (1180 TFLOP/s at
// kPoly 0 vs 1155 at 8, profiles/r1_attention_study.md), so MUFU only.
constexpr int kDefaultPoly = 0;
constexpr int kDefaultPChunks = 2;
constexpr int kDefaultSpec = 0;

}  // namespace

void attention_fwd(const AttnParams& p, cudaStream_t stream) {
  MRSP_REQUIRE(p.L > 0 && p.n_heads > 0 && p.q_per_kv > 0, MRSP_INVALID_ARGUMENT,
               "attention: empty problem");
  MRSP_REQUIRE(p.ldq % 8 == 0 && p.ldk % 8 == 0 && p.ldv % 8 == 0 && p.ldo % 8 == 0,
               MRSP_INVALID_ARGUMENT, "attention: leading dims must be multiples of 8");
  MRSP_REQUIRE(p.mode == ATTN_BLOCK_DIAG ? p.blk > 0 : (p.Lmax > 0 || p.Lp >= p.L),
               MRSP_INVALID_ARGUMENT, "attention: bad mask parameters");
  // kPoly (FMA-pipe share of the exp2s) is a tuning knob; MRSP_ATTN_POLY
  // overrides the default for sweeps (tools/attn_perf.py).
  // FMA-pipe exp2 share (MRSP_ATTN_POLY) is a tuning knob for sweeps
  // (tools/attn_perf.py); every instantiation is parity-tested.
  const char* env_poly = std::getenv("MRSP_ATTN_POLY");
  const int poly = env_poly ? std::atoi(env_poly) : kDefaultPoly;
  // MRSP_ATTN_PCHUNKS: 2 (64-key halves of P, default) or 4 (32-key quarters)
  const char* env_pc = std::getenv("MRSP_ATTN_PCHUNKS");
  const int pc = env_pc ? std::atoi(env_pc) : kDefaultPChunks;
  using Kern = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, AttnArgs);
  // MRSP_ATTN_SPEC: 1 speculative first-chunk exponentials (see kSpec), 0 max first
  const char* env_spec = std::getenv("MRSP_ATTN_SPEC");
  const int spec = env_spec ? std::atoi(env_spec) : kDefaultSpec;
  const Kern kern = spec ? (pc == 4 ? attn_fwd_tcgen05<0, 4, 1> : attn_fwd_tcgen05<0, 2, 1>)
                  : pc == 4 ? (poly == 8 ? attn_fwd_tcgen05<8, 4, 0> : attn_fwd_tcgen05<0, 4, 0>)
                  : poly == 4 ? attn_fwd_tcgen05<4, 2, 0> : poly == 8 ? attn_fwd_tcgen05<8, 2, 0>
                  : poly == 12 ? attn_fwd_tcgen05<12, 2, 0> : poly == 16 ? attn_fwd_tcgen05<16, 2, 0>
                  : attn_fwd_tcgen05<0, 2, 0>;
  static const bool attr = [] {
    for (auto k : {attn_fwd_tcgen05<0, 2, 0>, attn_fwd_tcgen05<4, 2, 0>, attn_fwd_tcgen05<8, 2, 0>,
                   attn_fwd_tcgen05<12, 2, 0>, attn_fwd_tcgen05<16, 2, 0>, attn_fwd_tcgen05<0, 4, 0>,
                   attn_fwd_tcgen05<8, 4, 0>, attn_fwd_tcgen05<0, 2, 1>, attn_fwd_tcgen05<0, 4, 1>})
      MRSP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(SMEM_BYTES)));
    return true;
  }();
  (void)attr;
  MRSP_REQUIRE(p.hstride == HD || (p.hstride > 0 && p.hstride < HD && p.hstride % 8 == 0 &&
                                   p.ldq % p.hstride == 0 && p.ldk % p.hstride == 0 &&
                                   p.ldv % p.hstride == 0 && p.q_col0 % p.hstride == 0 &&
                                   p.k_col0 % p.hstride == 0 && p.v_col0 % p.hstride == 0 &&
                                   p.n_dst == 0),
               MRSP_INVALID_ARGUMENT, "attention: head stride must be 128 or a multiple of 8 "
                                      "dividing the row pitches and column offsets");
  const bool h3 = p.hstride != HD;
  auto tmap = [&](const void* base, int ld, int box_rows) {
    return h3 ? make_tmap_bf16_3d_heads(base, p.L, ld / p.hstride, p.hstride, ld, box_rows, 64)
              : make_tmap_bf16_2d(base, p.L, ld, ld, box_rows, 64);
  };
  CUtensorMap tq = tmap(p.Q, p.ldq, TQ);
  CUtensorMap tk = tmap(p.K, p.ldk, TK);
  CUtensorMap tv = tmap(p.V, p.ldv, TK);
  AttnArgs a;
  const int n_q_tiles = (p.L + TQ - 1) / TQ;
  a.n_pairs = (n_q_tiles + 1) / 2;
  a.n_heads = p.n_heads;
  a.q_per_kv = p.q_per_kv;
  a.hs = p.hstride;
  a.q_col0 = h3 ? p.q_col0 / p.hstride : p.q_col0;
  a.k_col0 = h3 ? p.k_col0 / p.hstride : p.k_col0;
  a.v_col0 = h3 ? p.v_col0 / p.hstride : p.v_col0;
  a.o_col0 = p.o_col0;
  a.O = static_cast<__nv_bfloat16*>(p.O);
  a.ldo = p.ldo;
  a.scale_log2 = p.scale * 1.4426950408889634f;
  a.mask = MaskDev{p.mode, p.L, p.Lp, p.Lmax > 0 ? p.Lmax : 1, p.blk > 0 ? p.blk : 1};
  MRSP_REQUIRE(p.n_dst >= 0 && p.n_dst <= 8, MRSP_INVALID_ARGUMENT, "attention: <= 8 shards");
  a.n_dst = p.n_dst;
  a.dst_ld = p.dst_ld;
  a.dst_col0 = p.dst_col0;
  for (int i = 0; i < 9; ++i) a.dst_bounds[i] = p.dst_bounds[i];
  for (int i = 0; i < 8; ++i) a.dst_base[i] = static_cast<__nv_bfloat16*>(p.dst_base[i]);
  a.lse = p.lse;
  a.lse_ld = p.lse_ld;
  MRSP_REQUIRE(p.lse == nullptr || p.lse_ld >= p.L, MRSP_INVALID_ARGUMENT,
               "attention: lse row pitch shorter than L");
  MRSP_REQUIRE(p.row_parts >= 1 && p.row_part >= 0 && p.row_part < p.row_parts,
               MRSP_INVALID_ARGUMENT, "attention: bad query-row split");
  a.row_parts = p.row_parts;
  a.row_part = p.row_part;
  a.n_local = 0;
  while (a.row_parts == 1 ? a.n_local < a.n_pairs
                          : attn_row_block(a.n_local, a.row_part, a.n_pairs, a.row_parts) >= 0)
    ++a.n_local;
  if (a.n_local == 0) return;
  const int grid = a.n_local * a.n_heads;
  kern<<<grid, THREADS, SMEM_BYTES, stream>>>(tq, tk, tv, a);
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
