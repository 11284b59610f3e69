// decode.cu — the kernels of rollout generation: decode
// attention over the cached prompt prefix + each row's own generated keys,
// the split merge, and temperature sampling with the old log-prob.
//
// Decode attention (one generation step, G rows): per kv head, the q_per_kv x G
// queries (<= 64) attend to the shared prefix K/V (computed once by the prefix
// prefill, head-major [kv][K|V][Lp][128] per layer) and to the keys of their own row generated
// so far (time-major row cache [t][G][kv][128], row mask). The key range is
// split into chunks of DEC_CHUNK keys, one CTA per (chunk, kv head): each K/V
// tile read from HBM serves all of the kv group's queries (GQA reuse), and the
// CTA emits an unnormalised partial (m, l, O) merged by dec_merge_kernel —
// flash-decoding. Two implementations: the tcgen05 kernel (default; S, P, O in
// TMEM, TMA K/V ring, two KV streams per CTA for long prompts, an unmasked
// packed-FP32 softmax for full prompt tiles) and a register-blocked CUDA-core
// kernel (MRSP_DECODE_CC=1). Every kernel reads the step index from device
// memory, so a whole decode step is captured once as a CUDA graph
// (Engine::generate) and replayed for every t.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "common.h"
#include "misc.h"
#include "pdl.cuh"
#include "rownorm.cuh"
#include "sm100.cuh"
#include "tma.h"

namespace mrsp {
namespace {

constexpr int DEC_QN = 64;      // max queries per kv head (q_per_kv x G)
constexpr int DEC_KT = 64;      // keys per smem tile
constexpr int DEC_CHUNK = 512;  // keys per CTA
constexpr int HD = 128;

struct DecArgs {
  const __nv_bfloat16* q;  // [G][ldq] bf16, head h at column q_col0 + 128 h
  int ldq, q_col0;
  const __nv_bfloat16* kv_prefix;  // head-major [n_kv][K | V][Lp][128] (contiguous per head)
  const __nv_bfloat16* kv_rows;    // [(t+1) * G][ld_kv] time-major: row (s*G + g)
  int ld_kv, v_off;
  int Lp, G, q_per_kv, n_kv;
  const int* tdev;  // step index t (device)
  int n_prefix_chunks, n_row_chunks;
  float scale_log2;
  float* part;  // [n_chunks][n_kv][DEC_QN][HD + 2]
};

// Register-blocked CUDA-core flash-decoding tile loop. 256 threads; per 64-key
// tile: S[64 q][64 k] with a 4 q x 4 k block per thread (float4 smem loads
// along the head dim: 16 FMAs per 2 LDS.128), online softmax per query row
// (a row's 64 scores live in 16 lanes of one warp), then O[64 q][128 d] +=
// P.V with a 4 q x 8 d block per thread (32 FMAs per 3 LDS.128).
__global__ void __launch_bounds__(256)
    dec_attn_kernel(DecArgs a) {
  extern __shared__ __align__(16) float sm[];
  constexpr int QS = HD + 4;                  // padded row strides (floats)
  float* Qs = sm;                             // [DEC_QN][QS]
  float* Ks = Qs + DEC_QN * QS;               // [DEC_KT][QS]
  float* Vs = Ks + DEC_KT * QS;               // [DEC_KT][HD]
  float* Pt = Vs + DEC_KT * HD;               // [DEC_KT][DEC_QN]  (P transposed)
  float* row_alpha = Pt + DEC_KT * DEC_QN;    // [DEC_QN]
  const int chunk = blockIdx.x, kvh = blockIdx.y, tid = threadIdx.x;
  const int qn = a.q_per_kv * a.G;
  const bool rows_src = chunk >= a.n_prefix_chunks;
  const long k_begin = static_cast<long>(rows_src ? chunk - a.n_prefix_chunks : chunk) * DEC_CHUNK;
  const long k_total = rows_src ? static_cast<long>(*a.tdev + 1) * a.G : a.Lp;
  const long k_end = std::min<long>(k_begin + DEC_CHUNK, k_total);
  const __nv_bfloat16* src = rows_src ? a.kv_rows : a.kv_prefix;
  for (int i = tid; i < DEC_QN * HD; i += blockDim.x) {  // qi = hl * G + g
    const int qi = i / HD, d = i % HD;
    float v = 0.f;
    if (qi < qn) {
      const int hl = qi / a.G, g = qi % a.G;
      v = __bfloat162float(a.q[static_cast<size_t>(g) * a.ldq + a.q_col0 +
                               (kvh * a.q_per_kv + hl) * HD + d]);
    }
    Qs[qi * QS + d] = v * a.scale_log2;  // scores come out in the log2 domain
  }
  // S mapping: query block qb (4 rows) x keys kb + 16 c (c < 4): the 16 lanes
  // of a row group read 16 consecutive K rows (row stride 132 floats -> a
  // different 4-bank group per lane, no conflicts; 4 kb + c was 8-way)
  const int qb = tid >> 4, kb = tid & 15;
  // O mapping: query block ob (4 rows), head-dim block db (8 dims)
  const int ob = tid >> 4, db = tid & 15;
  float m_row[4], l_row[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    m_row[r] = -INFINITY;
    l_row[r] = 0.f;
  }
  float o[4][8];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int j = 0; j < 8; ++j) o[r][j] = 0.f;
  for (long k0 = k_begin; k0 < k_end; k0 += DEC_KT) {
    __syncthreads();
    for (int i = tid; i < DEC_KT * (HD / 8); i += blockDim.x) {  // 16-byte global loads
      const int kk = i / (HD / 8), c8 = (i % (HD / 8)) * 8;
      const long k = k0 + kk;
      uint4 ku = make_uint4(0, 0, 0, 0), vu = make_uint4(0, 0, 0, 0);
      if (k < k_end) {
        if (rows_src) {
          const __nv_bfloat16* row = src + static_cast<size_t>(k) * a.ld_kv;
          ku = *reinterpret_cast<const uint4*>(row + kvh * HD + c8);
          vu = *reinterpret_cast<const uint4*>(row + a.v_off + kvh * HD + c8);
        } else {
          const __nv_bfloat16* kr = src + (static_cast<size_t>(2 * kvh) * a.Lp + k) * HD;
          ku = *reinterpret_cast<const uint4*>(kr + c8);
          vu = *reinterpret_cast<const uint4*>(kr + static_cast<size_t>(a.Lp) * HD + c8);
        }
      }
      const __nv_bfloat162* k2 = reinterpret_cast<const __nv_bfloat162*>(&ku);
      const __nv_bfloat162* v2 = reinterpret_cast<const __nv_bfloat162*>(&vu);
      float4* kd = reinterpret_cast<float4*>(Ks + kk * QS + c8);
      float4* vd = reinterpret_cast<float4*>(Vs + kk * HD + c8);
      const float2 k01 = __bfloat1622float2(k2[0]), k23 = __bfloat1622float2(k2[1]);
      const float2 k45 = __bfloat1622float2(k2[2]), k67 = __bfloat1622float2(k2[3]);
      const float2 v01 = __bfloat1622float2(v2[0]), v23 = __bfloat1622float2(v2[1]);
      const float2 v45 = __bfloat1622float2(v2[2]), v67 = __bfloat1622float2(v2[3]);
      kd[0] = make_float4(k01.x, k01.y, k23.x, k23.y);
      kd[1] = make_float4(k45.x, k45.y, k67.x, k67.y);
      vd[0] = make_float4(v01.x, v01.y, v23.x, v23.y);
      vd[1] = make_float4(v45.x, v45.y, v67.x, v67.y);
    }
    __syncthreads();
    float sc[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) sc[r][c] = 0.f;
#pragma unroll 4
    for (int d = 0; d < HD; d += 4) {
      float4 qv[4], kv[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) qv[r] = *reinterpret_cast<const float4*>(Qs + (qb * 4 + r) * QS + d);
#pragma unroll
      for (int c = 0; c < 4; ++c) kv[c] = *reinterpret_cast<const float4*>(Ks + (kb + 16 * c) * QS + d);
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c)
          sc[r][c] = fmaf(qv[r].x, kv[c].x, fmaf(qv[r].y, kv[c].y,
                     fmaf(qv[r].z, kv[c].z, fmaf(qv[r].w, kv[c].w, sc[r][c]))));
    }
    // mask, online softmax per row (the row's 64 scores: 16 lanes x 4)
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int qi = qb * 4 + r;
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const long k = k0 + kb + 16 * c;
        bool vis = qi < qn && k < k_end;
        if (rows_src) vis = vis && static_cast<int>(k % a.G) == qi % a.G;  // own row only
        if (!vis) sc[r][c] = -INFINITY;
        mx = fmaxf(mx, sc[r][c]);
      }
#pragma unroll
      for (int off = 1; off < 16; off <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
      const float m_new = fmaxf(m_row[r], mx);
      const float alpha = m_new == -INFINITY ? 1.f : exp2f(m_row[r] - m_new);
      float ls = 0.f;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float p = m_new == -INFINITY ? 0.f : exp2f(sc[r][c] - m_new);
        Pt[(kb + 16 * c) * DEC_QN + qi] = p;
        ls += p;
      }
#pragma unroll
      for (int off = 1; off < 16; off <<= 1) ls += __shfl_xor_sync(0xffffffffu, ls, off);
      l_row[r] = l_row[r] * alpha + ls;
      m_row[r] = m_new;
      if (kb == 0) row_alpha[qi] = alpha;
    }
    __syncthreads();
    float al[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) al[r] = row_alpha[ob * 4 + r];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int j = 0; j < 8; ++j) o[r][j] *= al[r];
#pragma unroll 4
    for (int kk = 0; kk < DEC_KT; ++kk) {
      const float4 pv = *reinterpret_cast<const float4*>(Pt + kk * DEC_QN + ob * 4);
      const float4 v0 = *reinterpret_cast<const float4*>(Vs + kk * HD + db * 8);
      const float4 v1 = *reinterpret_cast<const float4*>(Vs + kk * HD + db * 8 + 4);
      const float pr[4] = {pv.x, pv.y, pv.z, pv.w};
      const float vv[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int j = 0; j < 8; ++j) o[r][j] = fmaf(pr[r], vv[j], o[r][j]);
    }
  }
  // partial (m, l, O): the S-mapping threads hold (m, l) of rows qb*4+r, the
  // O-mapping threads hold O of rows ob*4+r (same block index: qb == ob)
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int qi = ob * 4 + r;
    if (qi >= qn) continue;
    float* out = a.part + ((static_cast<size_t>(chunk) * a.n_kv + kvh) * DEC_QN + qi) * (HD + 2);
#pragma unroll
    for (int j = 0; j < 8; ++j) out[db * 8 + j] = o[r][j];
    if (db == 0) {
      out[HD] = m_row[r];
      out[HD + 1] = l_row[r];
    }
  }
}

// ---------------------------------------------------------------------------
// Tensor-core decode attention (the default): one CTA per (chunk, kv head),
// the <= 64 queries of the kv group as one 128-row Q tile (zero rows pad it)
// written to smem in the SW128 K-major layout, 128-key K/V tiles by TMA
// through a kRing-slot ring, S = Q.K^T and O += P.V on tcgen05 with S, P
// (bf16 over S) and O in TMEM — the prefill kernel's tile pipeline for one Q
// tile. Same unnormalised (m, l, O) partial as the CUDA-core kernel.
namespace tc {
using namespace sm100;
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
constexpr int TQ = 128, TK = 128, CHUNK = 128 * 64 * 2, TILE = 2 * CHUNK;
constexpr int OFF_Q = 0, OFF_RING = TILE;
// kRing = K/V ring slots: 2 (two CTAs per SM) or 6 (one CTA per SM, three
// tiles of K/V in flight so the HBM latency is off the per-tile chain)
template <int kRing>
constexpr size_t smem_bytes() { return 1024 + OFF_RING + kRing * TILE + 256; }

struct Args {
  const __nv_bfloat16* q;
  const int* tdev;  // step index t (device)
  int ldq, q_col0, G, Lp, q_per_kv, n_kv, n_prefix_chunks, chunk_keys;
  int v_off;
  float scale_log2;
  float* part;
};

// kStreams = 2 (one CTA per SM): the chunk's KV tiles alternate between two
// streams with their own S and O in TMEM (S0 S1 O0 O1 = 512 columns) and their
// own softmax warpgroup; the MMA issuer interleaves
//     S(0) S(1) | P.V(0) S(2) | P.V(1) S(3) | ...
// so one warpgroup's softmax overlaps the other stream's MMAs (the prefill
// kernel's ping-pong, over keys instead of query tiles). Each stream writes
// its own (m, l, O) partial (chunk slots 2c and 2c + 1; dec_merge_kernel
// combines them). kStreams = 1 (two CTAs per SM, short prompts): one stream.
template <int kStreams>
constexpr int threads() { return 128 + 128 * kStreams; }

constexpr float kDecRescale = 8.0f;  // log2 domain (lazy O rescale)

// Packed fp32x2 FMA / add (FFMA2 / FADD2): half the issue slots of the scalar forms.
__device__ __forceinline__ void dec_ffma2(float& d0, float& d1, float a0, float a1, float b0, float b1,
                                          float c0, float c1) {
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}
__device__ __forceinline__ void dec_fadd2(float& d0, float& d1, float a0, float a1) {
  asm("{\n\t.reg .b64 ra, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rd, {%0, %1};\n\t"
      "add.rn.f32x2 rd, rd, ra;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "+f"(d0), "+f"(d1)
      : "f"(a0), "f"(a1));
}

// Optional clock() timeline of CTA (0, 0) (tools/ubench/dec_trace.cu builds this
// file with MRSP_DEC_TRACE): lane 0 of each warp stamps (event, tile, clock).
#ifdef MRSP_DEC_TRACE
constexpr int kDecTraceCap = 4096;
__device__ uint64_t g_dec_trace[12][kDecTraceCap];
__device__ int g_dec_trace_n[12];
#define DTRACE(ev, j)                                                                          \
  do {                                                                                         \
    if (blockIdx.x == 0 && blockIdx.y == 0 && (threadIdx.x & 31) == 0 && dtn < kDecTraceCap) \
      g_dec_trace[threadIdx.x >> 5][dtn++] = (static_cast<uint64_t>(ev) << 56) |              \
                                             (static_cast<uint64_t>((j) & 0xffffff) << 32) |   \
                                             static_cast<uint32_t>(clock());                   \
  } while (0)
#define DTRACE_INIT int dtn = 0
#define DTRACE_FINISH \
  if (blockIdx.x == 0 && blockIdx.y == 0 && (threadIdx.x & 31) == 0) g_dec_trace_n[threadIdx.x >> 5] = dtn
#else
#define DTRACE(ev, j) \
  do {                \
  } while (0)
#define DTRACE_INIT
#define DTRACE_FINISH
#endif

template <int kRing, int kStreams>
__global__ void __launch_bounds__(threads<kStreams>(), kRing == 2 ? 2 : 1)
    dec_attn_tc_kernel(const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmR,
                       Args a) {
  constexpr int RING = kRing;
  constexpr uint32_t TMEM_COLS = 256 * kStreams;
  constexpr int OFF_BAR = OFF_RING + RING * TILE;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* q_ready = bars;
  uint64_t* r_full = bars + 1;        // [RING]
  uint64_t* r_empty = r_full + RING;  // [RING]
  uint64_t* s_full = r_empty + RING;  // [kStreams]
  uint64_t* p_full = s_full + kStreams;
  uint64_t* pv_done = p_full + kStreams;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + kStreams);
  const int warp = warp_id(), chunk = blockIdx.x, kvh = blockIdx.y;
  const int qn = a.q_per_kv * a.G;
  const bool rows_src = chunk >= a.n_prefix_chunks;
  const long k_begin = static_cast<long>(rows_src ? chunk - a.n_prefix_chunks : chunk) * a.chunk_keys;
  const long k_total = rows_src ? static_cast<long>(*a.tdev + 1) * a.G : a.Lp;
  const long k_end = std::min<long>(k_begin + a.chunk_keys, k_total);
  // chunks past the live row keys (graph replays size the grid for max_len) are empty
  const int n_tiles = k_end > k_begin ? static_cast<int>((k_end - k_begin + TK - 1) / TK) : 0;
  const CUtensorMap* tm = rows_src ? &tmR : &tmP;
  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(tm);
    mbar_init(q_ready, 128);
    for (int i = 0; i < RING; ++i) {
      mbar_init(&r_full[i], 1);
      mbar_init(&r_empty[i], 1);
    }
    for (int w = 0; w < kStreams; ++w) {
      mbar_init(&s_full[w], 1);
      mbar_init(&p_full[w], 128);
      mbar_init(&pv_done[w], 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // S_w at column 128 w (P over its first 64), O_w at 128 kStreams + 128 w
  const uint32_t tmem = *tmem_slot;
  // PDL (decode graphs): the prompt K/V (written by the prefill, long before)
  // streams in before pdl_wait(); Q, the row cache and the partials wait.
  pdl_trigger();
  DTRACE_INIT;
  DTRACE(0, 0);
  if (warp == 0) {
    if (elect_one()) {  // K_j, V_j alternate through the ring (ring item 2j, 2j + 1)
      int slot = 0;
      uint32_t ph = 0;
      bool waited = false;
      for (int j = 0; j < n_tiles; ++j)
        for (int kv = 0; kv < 2; ++kv) {
          if (!waited && (rows_src || 2 * j + kv >= RING)) {  // first slot reuse / row cache
            pdl_wait();
            waited = true;
          }
          mbar_wait(&r_empty[slot], ph ^ 1);
          DTRACE(1, 2 * j + kv);
          mbar_arrive_expect_tx(&r_full[slot], TILE);
          uint8_t* dst = smem + OFF_RING + slot * TILE;
          // row cache [rows][K heads | V heads]; prompt prefix head-major
          // [n_kv][K | V][Lp][128], so each box is 16 KB of contiguous HBM
          const int col = rows_src ? (kv ? a.v_off : 0) + kvh * 128 : 0;
          const int row = (rows_src ? 0 : (2 * kvh + kv) * a.Lp) + static_cast<int>(k_begin) + j * TK;
          tma_load_2d(dst, tm, &r_full[slot], col, row);
          tma_load_2d(dst + CHUNK, tm, &r_full[slot], col + 64, row);
          if (++slot == RING) { slot = 0; ph ^= 1; }
        }
    }
  } else if (warp == 1) {
    const uint32_t idesc_s = idesc_bf16_f32(TQ, TK), idesc_o = idesc_bf16_f32_bmn(TQ, 128);
    const uint32_t q_addr = smem_u32(smem + OFF_Q), ring = smem_u32(smem + OFF_RING);
    mbar_wait(q_ready, 0);
    tc_fence_after();
    // ring item i sits in slot i % RING, completion phase (i / RING) & 1
    auto issue_s = [&](int j) {  // S_{j % kStreams} = Q K_j^T
      const int item = 2 * j, slot = item % RING;
      DTRACE(2, j);
      mbar_wait(&r_full[slot], (item / RING) & 1);
      DTRACE(3, j);
      tc_fence_after();
      const uint32_t k_addr = ring + slot * TILE;
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk / 4) * CHUNK + (kk % 4) * 32;
          mma_bf16_ss(tmem + (j % kStreams) * 128, sdesc_sw128(q_addr + off), sdesc_sw128(k_addr + off),
                      idesc_s, kk > 0 ? 1u : 0u);
        }
        mma_commit(&s_full[j % kStreams]);
        mma_commit(&r_empty[slot]);
      }
      __syncwarp();
    };
    auto issue_pv = [&](int j) {  // O_{j % kStreams} += P_j V_j
      const int w = j % kStreams, item = 2 * j + 1, slot = item % RING;
      DTRACE(4, j);
      mbar_wait(&p_full[w], (j / kStreams) & 1);
      DTRACE(5, j);
      mbar_wait(&r_full[slot], (item / RING) & 1);
      DTRACE(6, j);
      tc_fence_after();
      const uint32_t v_addr = ring + slot * TILE;
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_bf16_ts(tmem + 128 * kStreams + 128 * w, tmem + w * 128 + kk * 8,
                      sdesc_sw128_mn(v_addr + kk * 2048, CHUNK), idesc_o,
                      (j >= kStreams || kk > 0) ? 1u : 0u);
        mma_commit(&pv_done[w]);
        mma_commit(&r_empty[slot]);
      }
      __syncwarp();
    };
    for (int j = 0; j < kStreams && j < n_tiles; ++j) issue_s(j);
    for (int j = 0; j < n_tiles; ++j) {
      issue_pv(j);  // P_j is read before S_{j + kStreams} overwrites it (in-order MMAs)
      if (j + kStreams < n_tiles) issue_s(j + kStreams);
    }
  } else if (warp >= 4) {
    const int w = (warp - 4) >> 2;                    // stream of this warpgroup
    const int r = ((warp - 4) & 3) * 32 + lane_id();  // query row = TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>(((warp - 4) & 3) * 32) << 16;
    const uint32_t tS = tmem + lane_off + 128 * w, tO = tmem + lane_off + 128 * kStreams + 128 * w;
    pdl_wait();  // Q and (epilogue) the partials depend on / are read by earlier kernels
    if (w == 0) {  // Q row r -> smem, SW128 K-major: 16-byte unit u of a 128-byte row at u ^ (r & 7)
      uint4 v[16];
      if (r < qn) {
        const int hl = r / a.G, g = r % a.G;
        const uint4* src = reinterpret_cast<const uint4*>(
            a.q + static_cast<size_t>(g) * a.ldq + a.q_col0 + (kvh * a.q_per_kv + hl) * 128);
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = src[u];
      } else {
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int half = u / 8, uu = u % 8;
        *reinterpret_cast<uint4*>(smem + OFF_Q + half * CHUNK + r * 128 + ((uu ^ (r & 7)) * 16)) = v[u];
      }
      fence_proxy_async_smem();
      mbar_arrive(q_ready);
    }
    const int g_of_r = r % a.G;
    float m_run = -INFINITY, l_run = 0.f;
    int it = 0;  // tiles of this stream
    // two passes over S in TMEM (32 columns at a time, <= 128 registers per
    // thread so two CTAs share an SM): row max, then exp / P / row sum.
    // Visibility is one 32-bit mask per 32 keys, built once per tile: keys
    // below the chunk end, and (row cache) only this query's own rollout row.
    for (int j = w; j < n_tiles; j += kStreams, ++it) {
      mbar_wait(&s_full[w], it & 1);
      DTRACE(7, j);
      tc_fence_after();
      const long k0 = k_begin + static_cast<long>(j) * TK;
      // full prompt tile: every row sees all 128 keys (rows >= qn are padding
      // whose results are never stored), so no element mask — warp-uniform
      const bool full = !rows_src && k0 + TK <= k_end;
      uint32_t vis[4] = {~0u, ~0u, ~0u, ~0u};
      if (!full) {
        const int nv = r < qn ? static_cast<int>(std::min<long>(TK, k_end - k0)) : 0;
        const int o = rows_src ? static_cast<int>(((g_of_r - k0 % a.G) % a.G + a.G) % a.G) : 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int n = nv - 32 * q;
          uint32_t m = n <= 0 ? 0u : (n >= 32 ? 0xffffffffu : (1u << n) - 1u);
          if (rows_src) {  // key k0 + 32 q + i is row (k0 + 32 q + i) % G
            uint32_t rm = 0;
            for (int i = (o - 32 * q % a.G + a.G) % a.G; i < 32; i += a.G) rm |= 1u << i;
            m &= rm;
          }
          vis[q] = m;
        }
      }
      float mx = -INFINITY;
      if (full) {  // max of the raw scores (scale > 0), two independent FMNMX3 chains
        float m2[2] = {-INFINITY, -INFINITY};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t x[32];
          tmem_ld32(tS + 32 * q, x);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; i += 2)
            m2[(i >> 1) & 1] = fmaxf(m2[(i >> 1) & 1], fmaxf(__uint_as_float(x[i]), __uint_as_float(x[i + 1])));
        }
        mx = fmaxf(m2[0], m2[1]) * a.scale_log2;
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t x[32];
          tmem_ld32(tS + 32 * q, x);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i)
            mx = fmaxf(mx, (vis[q] >> i) & 1u ? __uint_as_float(x[i]) * a.scale_log2 : -INFINITY);
        }
      }
      // lazy rescale (as the prefill kernel): O and l are rescaled only when a
      // row's max grows by more than 2^8; P = 2^(s - m_run) <= 2^8 otherwise
      const float m_new = fmaxf(m_run, mx);
      const bool need = m_new > m_run + kDecRescale;
      if (it > 0 && __any_sync(0xffffffffu, need)) {  // rescale O_w (after its last P.V)
        mbar_wait(&pv_done[w], (it - 1) & 1);
        tc_fence_after();
        const float alpha = need && m_run != -INFINITY ? exp2f(m_run - m_new) : 1.f;
#pragma unroll 1
        for (int c = 0; c < 128; c += 32) {
          uint32_t o[32];
          tmem_ld32(tO + c, o);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          tmem_st32(tO + c, o);
        }
        tmem_st_wait();
        l_run *= alpha;
      }
      if (need) m_run = m_new;
      const float nm = m_run == -INFINITY ? 0.f : -m_run;
      const float sl = a.scale_log2;
      float acc = 0.f;
      if (full) {  // packed fp32x2 FMA / add, 8 partial sums
        float ac[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          uint32_t wv[32];
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            uint32_t x[32];
            tmem_ld32(tS + h * 64 + cc * 32, x);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
              float y0, y1;
              dec_ffma2(y0, y1, __uint_as_float(x[i]), __uint_as_float(x[i + 1]), sl, sl, nm, nm);
              const float p0 = ex2_approx(y0), p1 = ex2_approx(y1);
              const int q = ((i >> 1) & 3) * 2;
              dec_fadd2(ac[q], ac[q + 1], p0, p1);
              wv[cc * 16 + i / 2] = pack_bf16(p0, p1);
            }
          }
          tmem_st32(tS + 32 * h, wv);
        }
        acc = ((ac[0] + ac[1]) + (ac[2] + ac[3])) + ((ac[4] + ac[5]) + (ac[6] + ac[7]));
      } else {
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {  // 64-key halves: P(half h) -> columns [32 h, 32 h + 32),
          uint32_t wv[32];              // over S columns whose keys are already consumed
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            const int c = h * 64 + cc * 32;
            uint32_t x[32];
            tmem_ld32(tS + c, x);
            tmem_ld_wait();
            const uint32_t vm = vis[c / 32];
#pragma unroll
            for (int i = 0; i < 32; i += 2) {  // ex2(-inf) = 0 for masked keys
              const float p0 = ex2_approx((vm >> i) & 1u ? fmaf(__uint_as_float(x[i]), sl, nm) : -INFINITY);
              const float p1 =
                  ex2_approx((vm >> (i + 1)) & 1u ? fmaf(__uint_as_float(x[i + 1]), sl, nm) : -INFINITY);
              acc += p0 + p1;
              wv[cc * 16 + i / 2] = pack_bf16(p0, p1);
            }
          }
          tmem_st32(tS + 32 * h, wv);
        }
      }
      tmem_st_wait();
      l_run += acc;
      tc_fence_before();
      mbar_arrive(&p_full[w]);
      DTRACE(8, j);
    }
    // epilogue: the unnormalised partial of this stream of the chunk
    if (it > 0) {
      mbar_wait(&pv_done[w], (it - 1) & 1);
      tc_fence_after();
    }
    float* out = a.part +
                 ((static_cast<size_t>(chunk * kStreams + w) * a.n_kv + kvh) * DEC_QN + r) * (HD + 2);
#pragma unroll 1
    for (int c = 0; c < 128; c += 32) {
      uint32_t o[32];
      tmem_ld32(tO + c, o);
      tmem_ld_wait();
      if (r < qn)
#pragma unroll
        for (int i = 0; i < 32; ++i) out[c + i] = it > 0 ? __uint_as_float(o[i]) : 0.f;
    }
    if (r < qn) {
      out[HD] = it > 0 ? m_run : -INFINITY;
      out[HD + 1] = l_run;
    }
  }
  DTRACE(9, 0);
  DTRACE_FINISH;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<TMEM_COLS>(tmem);
}
}  // namespace tc

// O[g][h*128 + d] = sum_c O_c 2^(m_c - m) / sum_c l_c 2^(m_c - m). The chunk
// maxima and weights are formed by all threads at once (smem); four groups of
// 128 threads (one per column) sum every fourth chunk with the loads unrolled,
// and the four group sums are added in group order (deterministic). Empty
// chunks (m_c = -inf) carry weight 0 and zero partials.
constexpr int kMergeMaxChunks = 1024, kMergeGroups = 4;
__global__ void __launch_bounds__(HD * kMergeGroups)
    dec_merge_kernel(const float* __restrict__ part, int n_chunks, int n_kv, int q_per_kv, int G,
                     __nv_bfloat16* __restrict__ out, int ldo) {
  pdl_wait();
  pdl_trigger();
  __shared__ float s_w[kMergeMaxChunks], s_l[kMergeMaxChunks], s_red[HD * kMergeGroups / 32];
  __shared__ float s_o[kMergeGroups][HD], s_lg[kMergeGroups];
  const int qi = blockIdx.x, kvh = blockIdx.y, tid = threadIdx.x;
  const int d = tid % HD, grp = tid / HD;
  const int hl = qi / G, g = qi % G;
  auto row = [&](int c) {
    return part + ((static_cast<size_t>(c) * n_kv + kvh) * DEC_QN + qi) * (HD + 2);
  };
  float m = -INFINITY;
  for (int c = tid; c < n_chunks; c += blockDim.x) {
    const float mc = row(c)[HD];
    s_w[c] = mc;
    s_l[c] = row(c)[HD + 1];
    m = fmaxf(m, mc);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((tid & 31) == 0) s_red[tid >> 5] = m;
  __syncthreads();
  m = -INFINITY;
#pragma unroll
  for (int i = 0; i < HD * kMergeGroups / 32; ++i) m = fmaxf(m, s_red[i]);
  for (int c = tid; c < n_chunks; c += blockDim.x) s_w[c] = s_w[c] == -INFINITY ? 0.f : exp2f(s_w[c] - m);
  __syncthreads();
  float lg = 0.f, og = 0.f;
  int c = grp;
  for (; c + 3 * kMergeGroups < n_chunks; c += 4 * kMergeGroups) {
    float v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = row(c + u * kMergeGroups)[d];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      lg += s_l[c + u * kMergeGroups] * s_w[c + u * kMergeGroups];
      og += v[u] * s_w[c + u * kMergeGroups];
    }
  }
  for (; c < n_chunks; c += kMergeGroups) {
    lg += s_l[c] * s_w[c];
    og += row(c)[d] * s_w[c];
  }
  s_o[grp][d] = og;
  if (d == 0) s_lg[grp] = lg;
  __syncthreads();
  if (grp != 0) return;
  float l = 0.f, o = 0.f;
#pragma unroll
  for (int k = 0; k < kMergeGroups; ++k) {
    l += s_lg[k];
    o += s_o[k][d];
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

// Sampling, p = softmax(logits / T); token = first v with cdf(v) > u,
// u = (splitmix64(seed, row, t) >> 11) * 2^-53 * Z; old_lp = log_softmax(logits)[token]
// at temperature 1 (policy.cpp:130-134). Rows already finished (EOS) only
// record PAD. fp64 accumulation. Two kernels so the vocabulary sweep spreads
// over the SMs: sample_slices_kernel (grid kSampleSlices x G) reduces each
// vocabulary slice to (max, sum exp((x - max) / T), sum exp(x - max)), and
// sample_pick_kernel (one CTA per row) combines the slices in slice order,
// finds the slice holding u, and walks only that slice.
constexpr int kSampleSlices = 16;

template <typename T>
__device__ __forceinline__ T block_reduce(T v, T* red, bool is_max) {
  const int tid = threadIdx.x, nw = blockDim.x >> 5;
  for (int o = 16; o; o >>= 1) {
    const T w = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? (v > w ? v : w) : v + w;
  }
  if ((tid & 31) == 0) red[tid >> 5] = v;
  __syncthreads();
  if (tid < 32) {
    v = tid < nw ? red[tid] : (is_max ? static_cast<T>(-INFINITY) : static_cast<T>(0));
    for (int o = 16; o; o >>= 1) {
      const T w = __shfl_xor_sync(0xffffffffu, v, o);
      v = is_max ? (v > w ? v : w) : v + w;
    }
    if (tid == 0) red[0] = v;
  }
  __syncthreads();
  const T r = red[0];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(256)
    sample_slices_kernel(const float* __restrict__ logits, int V, float inv_temp,
                         const int* __restrict__ done, double* __restrict__ part) {
  pdl_wait();
  pdl_trigger();
  const int sl = blockIdx.x, g = blockIdx.y, tid = threadIdx.x;
  if (done[g]) return;
  __shared__ float redf[32];
  __shared__ double red[32];
  const int v0 = static_cast<int>(static_cast<long>(V) * sl / kSampleSlices);
  const int v1 = static_cast<int>(static_cast<long>(V) * (sl + 1) / kSampleSlices);
  const float* x = logits + static_cast<size_t>(g) * V;
  float mx = -INFINITY;
  for (int v = v0 + tid; v < v1; v += blockDim.x) mx = fmaxf(mx, x[v]);
  mx = block_reduce<float>(mx, redf, true);
  double zs = 0.0, z1 = 0.0;
  for (int v = v0 + tid; v < v1; v += blockDim.x) {
    const double d = static_cast<double>(x[v]) - mx;
    zs += exp(d * inv_temp);
    z1 += exp(d);
  }
  zs = block_reduce<double>(zs, red, false);
  z1 = block_reduce<double>(z1, red, false);
  if (tid == 0) {
    double* p = part + (static_cast<size_t>(g) * kSampleSlices + sl) * 3;
    p[0] = mx;
    p[1] = zs;
    p[2] = z1;
  }
}

__global__ void __launch_bounds__(1024)
    sample_pick_kernel(const float* __restrict__ logits, int V, float inv_temp, uint64_t seed,
                       const int* __restrict__ tdev, const double* __restrict__ part,
                       int* __restrict__ done, int* __restrict__ tokens, float* __restrict__ old_lp,
                       int* __restrict__ lengths, int max_len, int eos, int pad) {
  pdl_wait();
  pdl_trigger();
  const int g = blockIdx.x, tid = threadIdx.x, nt = blockDim.x, t = *tdev;
  __shared__ double red[32];
  __shared__ double s_cum[kSampleSlices];
  __shared__ int pick, s_slice;
  __shared__ double s_base, s_m, s_z1;
  if (done[g]) {
    if (tid == 0) tokens[static_cast<size_t>(g) * max_len + t] = pad;
    return;
  }
  const float* x = logits + static_cast<size_t>(g) * V;
  const double* p = part + static_cast<size_t>(g) * kSampleSlices * 3;
  if (tid == 0) {  // combine the slices in slice order
    double m = -INFINITY;
    for (int s = 0; s < kSampleSlices; ++s) m = fmax(m, p[3 * s]);
    double zs = 0.0, z1 = 0.0;
    for (int s = 0; s < kSampleSlices; ++s) {
      zs += p[3 * s + 1] * exp((p[3 * s] - m) * inv_temp);
      z1 += p[3 * s + 2] * exp(p[3 * s] - m);
      s_cum[s] = zs;
    }
    const double u = static_cast<double>(mix64(seed ^ mix64((static_cast<uint64_t>(g) << 32) |
                                                           static_cast<uint32_t>(t))) >> 11) *
                     0x1.0p-53 * zs;
    int sl = kSampleSlices - 1;
    for (int s = 0; s < kSampleSlices; ++s)
      if (u < s_cum[s]) {
        sl = s;
        break;
      }
    s_slice = sl;
    s_base = u - (sl ? s_cum[sl - 1] : 0.0);  // u relative to the slice start
    s_m = m;
    s_z1 = z1;
  }
  __syncthreads();
  const int sl = s_slice;
  const double m = s_m, u = s_base;
  const int v0s = static_cast<int>(static_cast<long>(V) * sl / kSampleSlices);
  const int v1s = static_cast<int>(static_cast<long>(V) * (sl + 1) / kSampleSlices);
  // inverse CDF inside the slice: each thread owns a contiguous piece; an
  // exclusive scan of the piece sums finds the piece containing u, then that
  // thread walks it
  const int per = (v1s - v0s + nt - 1) / nt, v0 = v0s + tid * per, v1 = min(v1s, v0 + per);
  double mine = 0.0;
  for (int v = v0; v < v1; ++v) mine += exp((static_cast<double>(x[v]) - m) * inv_temp);
  double inc = mine;
  for (int o = 1; o < 32; o <<= 1) {
    const double n = __shfl_up_sync(0xffffffffu, inc, o);
    if ((tid & 31) >= o) inc += n;
  }
  if ((tid & 31) == 31) red[tid >> 5] = inc;
  if (tid == 0) pick = v1s - 1;
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
  if (v0 < v1 && u >= before && u < before + mine) {
    double c = before;
    int chosen = v1 - 1;
    for (int v = v0; v < v1; ++v) {
      c += exp((static_cast<double>(x[v]) - m) * inv_temp);
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
        static_cast<float>(static_cast<double>(x[tok]) - m - log(s_z1));
    lengths[g] = t + 1;
    if (tok == eos) done[g] = 1;
  }
}

// hidden[g] = embed[prev token of row g] (EOS at t = 0, policy.cpp:127), and
// the position id Lp + t of every row (rows restart at Lp, as in the pack).
__global__ void decode_embed_kernel(const __nv_bfloat16* __restrict__ embed, int d,
                                    const int* __restrict__ tokens, int max_len,
                                    const int* __restrict__ tdev, int pos_base,
                                    float* __restrict__ hidden, int* __restrict__ pos_out,
                                    const float* __restrict__ norm_w,
                                    __nv_bfloat16* __restrict__ norm_out, float eps) {
  pdl_wait();
  pdl_trigger();
  const int g = blockIdx.x, t = *tdev, pos = pos_base + t;
  const int tok = t == 0 ? 1 /* Vocab::kEos */ : tokens[static_cast<size_t>(g) * max_len + t - 1];
  if (threadIdx.x == 0) pos_out[g] = pos;
  const __nv_bfloat162* src = reinterpret_cast<const __nv_bfloat162*>(embed + static_cast<size_t>(tok) * d);
  float2* dst = reinterpret_cast<float2*>(hidden + static_cast<size_t>(g) * d);
  for (int i = threadIdx.x; i < d / 2; i += blockDim.x) dst[i] = __bfloat1622float2(src[i]);
  if (norm_w) {  // fused first RMSNorm of the step (rmsnorm_kernel's bits)
    __syncthreads();
    block_rmsnorm_row(hidden + static_cast<size_t>(g) * d, norm_w, norm_out + static_cast<size_t>(g) * d,
                      d, eps);
  }
}

// rows[t * G + g] = qkv[g][col0, col0 + kvw): this step's post-RoPE K and V
// of every rollout row into the row cache, at the device-side step index.
__global__ void decode_append_kv_kernel(const __nv_bfloat16* __restrict__ qkv, int ldq, int col0,
                                        __nv_bfloat16* __restrict__ rows, int kvw,
                                        const int* __restrict__ tdev) {
  pdl_wait();
  pdl_trigger();
  const int g = blockIdx.x, G = gridDim.x;
  const uint4* src = reinterpret_cast<const uint4*>(qkv + static_cast<size_t>(g) * ldq + col0);
  uint4* dst = reinterpret_cast<uint4*>(rows + (static_cast<size_t>(*tdev) * G + g) * kvw);
  for (int i = threadIdx.x; i < kvw / 8; i += blockDim.x) dst[i] = src[i];
}

__global__ void decode_step_advance_kernel(int* tdev) {
  pdl_wait();
  if (threadIdx.x == 0) *tdev += 1;
}

}  // namespace

void decode_embed(const __nv_bfloat16* embed, int d, const int* tokens, int max_len,
                  const int* tdev, int G, int pos_base, float* hidden, int* pos_out, cudaStream_t s,
                  const float* norm_w, __nv_bfloat16* norm_out, float eps) {
  MRSP_REQUIRE(d % 4 == 0, MRSP_INVALID_ARGUMENT, "decode_embed: d % 4");
  launch_pdl(decode_embed_kernel, dim3(G), dim3(256), 0, s, embed, d, tokens, max_len, tdev, pos_base,
             hidden, pos_out, norm_w, norm_out, eps);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

void decode_append_kv(const __nv_bfloat16* qkv, int ldq, int col0, __nv_bfloat16* rows, int kvw,
                      int G, const int* tdev, cudaStream_t s) {
  MRSP_REQUIRE(kvw % 8 == 0 && ldq % 8 == 0 && col0 % 8 == 0, MRSP_INVALID_ARGUMENT,
               "decode_append_kv: 16-byte aligned rows");
  launch_pdl(decode_append_kv_kernel, dim3(G), dim3(128), 0, s, qkv, ldq, col0, rows, kvw, tdev);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

void decode_step_advance(int* tdev, cudaStream_t s) {
  launch_pdl(decode_step_advance_kernel, dim3(1), dim3(32), 0, s, tdev);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

size_t decode_partial_bytes(int max_prefix, int max_len, int G, int n_kv) {
  const int chunks = (max_prefix + DEC_CHUNK - 1) / DEC_CHUNK +
                     (max_len * G + DEC_CHUNK - 1) / DEC_CHUNK;
  // x 2: the tcgen05 kernel writes one partial per KV stream (two per chunk)
  return 2 * static_cast<size_t>(chunks) * n_kv * DEC_QN * (HD + 2) * sizeof(float);
}

// Kernel choice: the tcgen05 kernel (attention 2.0-2.4 ms per c4 decode step,
// 0.18 ms at c2) beats the register-blocked CUDA-core one (10+ / 0.61 ms) at
// every prompt length measured; MRSP_DECODE_CC=1 selects the CUDA-core kernel.
bool decode_use_tensor_cores(int Lp) {
  (void)Lp;
  const char* e = std::getenv("MRSP_DECODE_CC");
  return !(e && std::atoi(e) != 0);
}

void decode_tensor_maps(const void* kv_prefix, int Lp, int n_kv, const void* kv_rows, long rows,
                        int ld_kv, void* maps_out) {
  CUtensorMap* m = static_cast<CUtensorMap*>(maps_out);
  m[0] = make_tmap_bf16_2d(kv_prefix, static_cast<uint64_t>(2 * n_kv) * std::max(Lp, 1), 128, 128,
                           128, 64);
  m[1] = make_tmap_bf16_2d(kv_rows, std::max<long>(rows, 1), ld_kv, ld_kv, 128, 64);
}

void decode_attention(const void* q, int ldq, int q_col0, const void* kv_prefix,
                      const void* kv_rows, int ld_kv, int v_off, int Lp, int G, int t_grid,
                      int max_rows, const int* tdev, int q_per_kv, int n_kv, float scale,
                      float* part, void* out, int ldo, cudaStream_t s, const void* maps) {
  const int t = t_grid;
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
  a.tdev = tdev;
  a.q_per_kv = q_per_kv;
  a.n_kv = n_kv;
  a.n_prefix_chunks = (Lp + DEC_CHUNK - 1) / DEC_CHUNK;
  a.n_row_chunks = ((t + 1) * G + DEC_CHUNK - 1) / DEC_CHUNK;
  a.scale_log2 = scale * 1.4426950408889634f;
  a.part = part;
  if (decode_use_tensor_cores(Lp)) {
    tc::Args ta;
    ta.q = a.q;
    ta.ldq = ldq;
    ta.q_col0 = q_col0;
    ta.G = G;
    ta.tdev = tdev;
    ta.Lp = Lp;
    ta.q_per_kv = q_per_kv;
    ta.n_kv = n_kv;
    ta.v_off = v_off;
    ta.scale_log2 = a.scale_log2;
    ta.part = part;
    static const bool tc_attr = [] {
      MRSP_CUDA(cudaFuncSetAttribute(tc::dec_attn_tc_kernel<2, 1>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(tc::smem_bytes<2>())));
      MRSP_CUDA(cudaFuncSetAttribute(tc::dec_attn_tc_kernel<6, 1>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(tc::smem_bytes<6>())));
      MRSP_CUDA(cudaFuncSetAttribute(tc::dec_attn_tc_kernel<6, 2>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(tc::smem_bytes<6>())));
      return true;
    }();
    (void)tc_attr;
    const char* env_ring = std::getenv("MRSP_DECODE_RING");
    // long prompts: one CTA per SM with 3 tiles of K/V in flight (c4: 1.6-1.8
    // vs 2.2-2.8 ms per step); short ones: two CTAs per SM (c2: 0.12 vs 0.17)
    const int ring = env_ring ? std::atoi(env_ring) : (Lp >= 32768 ? 6 : 2);
    {  // chunks sized so that n_kv x (prompt chunks + row-cache chunks) fits in
       // one wave (2 or 1 resident CTAs per SM): a second wave of a few full
       // chunks would double the kernel's time
      const int per_kv = std::max(1, (ring == 2 ? 2 : 1) * num_sms() / n_kv);
      const long row_keys = static_cast<long>(max_rows);  // independent of t: eager = graph bits
      int ck = std::max(512, (Lp + per_kv - 1) / per_kv);
      ck = (ck + tc::TK - 1) / tc::TK * tc::TK;
      while ((Lp + ck - 1) / ck + (row_keys + ck - 1) / ck > per_kv) ck += tc::TK;
      ta.chunk_keys = ck;
      ta.n_prefix_chunks = (Lp + ta.chunk_keys - 1) / ta.chunk_keys;
    }
    // prompt K|V [Lp][ld_kv] and the row cache as TMA tensors (rows past the
    // current step are masked; the caller's row cache is zero-initialised)
    CUtensorMap tm[2];
    if (maps)
      std::memcpy(tm, maps, sizeof(tm));
    else
      decode_tensor_maps(kv_prefix, Lp, n_kv, kv_rows, static_cast<long>(t + 1) * G, ld_kv, tm);
    const int chunks = ta.n_prefix_chunks + ((t + 1) * G + ta.chunk_keys - 1) / ta.chunk_keys;
    // one CTA per SM: two KV streams per CTA (MRSP_DECODE_STREAMS=1: one)
    const char* env_streams = std::getenv("MRSP_DECODE_STREAMS");
    const int streams = ring == 2 ? 1 : (env_streams ? std::max(1, std::min(2, std::atoi(env_streams))) : 2);
    if (ring == 2)
      launch_pdl(tc::dec_attn_tc_kernel<2, 1>, dim3(chunks, n_kv), dim3(tc::threads<1>()),
                 tc::smem_bytes<2>(), s, tm[0], tm[1], ta);
    else if (streams == 1)
      launch_pdl(tc::dec_attn_tc_kernel<6, 1>, dim3(chunks, n_kv), dim3(tc::threads<1>()),
                 tc::smem_bytes<6>(), s, tm[0], tm[1], ta);
    else
      launch_pdl(tc::dec_attn_tc_kernel<6, 2>, dim3(chunks, n_kv), dim3(tc::threads<2>()),
                 tc::smem_bytes<6>(), s, tm[0], tm[1], ta);
    count_launch();
    MRSP_CUDA(cudaGetLastError());
    MRSP_REQUIRE(chunks * streams <= kMergeMaxChunks, MRSP_INVALID_ARGUMENT,
                 "decode attention: too many key chunks");
    launch_pdl(dec_merge_kernel, dim3(q_per_kv * G, n_kv), dim3(HD * kMergeGroups), 0, s, part,
               chunks * streams,
               n_kv, q_per_kv, G, static_cast<__nv_bfloat16*>(out), ldo);
    count_launch();
    MRSP_CUDA(cudaGetLastError());
    return;
  }
  const size_t smem =
      (DEC_QN * (HD + 4) + DEC_KT * (HD + 4) + DEC_KT * HD + DEC_KT * DEC_QN + DEC_QN) * sizeof(float);
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
  MRSP_REQUIRE(chunks <= kMergeMaxChunks, MRSP_INVALID_ARGUMENT, "decode attention: too many key chunks");
  dec_merge_kernel<<<dim3(q_per_kv * G, n_kv), HD * kMergeGroups, 0, s>>>(part, chunks, n_kv, q_per_kv, G,
                                                           static_cast<__nv_bfloat16*>(out), ldo);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

size_t sample_workspace_bytes(int G) { return static_cast<size_t>(G) * kSampleSlices * 3 * sizeof(double); }

void sample_tokens(const float* logits, int G, int V, float temperature, uint64_t seed,
                   const int* tdev, int* done, int* tokens, float* old_lp, int* lengths,
                   int max_len, void* ws, cudaStream_t s) {
  MRSP_REQUIRE(V >= kSampleSlices, MRSP_INVALID_ARGUMENT, "sample: vocabulary smaller than the slices");
  double* part = static_cast<double*>(ws);
  launch_pdl(sample_slices_kernel, dim3(kSampleSlices, G), dim3(256), 0, s, logits, V,
             1.0f / temperature, done, part);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
  launch_pdl(sample_pick_kernel, dim3(G), dim3(1024), 0, s, logits, V, 1.0f / temperature, seed, tdev,
             part, done, tokens, old_lp, lengths, max_len, /*Vocab::kEos*/ 1, /*Vocab::kPad*/ 0);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

}  // namespace mrsp
