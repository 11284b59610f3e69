// attn_common.cuh — pieces shared by the tcgen05 attention forward
// (attention.cu) and backward (backward.cu) kernels: the MR-SP mask tile
// classification, packed fp32x2 arithmetic, MUFU exp2, visibility bitmasks
// and the setmaxnreg register rebalancing.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "attention.h"
#include "mrsp_c.h"

namespace mrsp {
namespace attn_detail {

constexpr int TQ = 128, TK = 128, HD = 128;

struct MaskDev {
  int mode, L, Lp, Lmax, blk;
};

__device__ __forceinline__ int seg_of(int x, const MaskDev& m) { return (x - m.Lp) / m.Lmax; }

// 0 = skip, 1 = fully visible, 2 = needs the element mask.
__device__ __forceinline__ int tile_class(int q0, int kt, const MaskDev& m) {
  const int k0 = kt * TK, klast = k0 + TK - 1, qlast = q0 + TQ - 1;
  if (k0 >= m.L || q0 >= m.L) return 0;
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

// Packed fp32x2 FMA / add / sub (FFMA2 / FADD2 on sm_100a): half the issue slots.
__device__ __forceinline__ void ffma2(float& d0, float& d1, float a0, float a1, float b0, float b1,
                                      float c0, float c1) {
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}
__device__ __forceinline__ void fadd2(float& d0, float& d1, float a0, float a1) {
  asm("{\n\t.reg .b64 ra, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rd, {%0, %1};\n\t"
      "add.rn.f32x2 rd, rd, ra;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "+f"(d0), "+f"(d1)
      : "f"(a0), "f"(a1));
}
__device__ __forceinline__ void fsub2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "sub.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}

__device__ __forceinline__ void fmul2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}

// (2^x0, 2^x1) on the FMA pipe, packed: x = j + f with j = round(x) taken from
// the low mantissa bits of x + 1.5*2^23, f in [-0.5, 0.5], degree-3 minimax
// polynomial for 2^f (max rel. error 7.7e-5, far below bf16's 3.9e-3), then j
// added to the exponent field (one LEA). 8 issue slots per pair instead of two
// MUFU.EX2 (which is the softmax's binding pipe: 16 results/clk/SM, the same
// rate the tensor core consumes P at). Inputs clamp at -126 (2^-126 ~ 1e-38,
// i.e. zero after the P.V product and the row sum).
__device__ __forceinline__ void exp2_poly2(float x0, float x1, float& p0, float& p1) {
  constexpr float kRound = 12582912.0f;  // 1.5 * 2^23
  x0 = fmaxf(x0, -126.0f);
  x1 = fmaxf(x1, -126.0f);
  float r0 = x0, r1 = x1;
  fadd2(r0, r1, kRound, kRound);
  float t0, t1, f0, f1;
  fsub2(t0, t1, r0, r1, kRound, kRound);
  fsub2(f0, f1, x0, x1, t0, t1);
  float q0, q1;
  ffma2(q0, q1, f0, f1, 0.05508868396282196f, 0.05508868396282196f, 0.24260404706001282f,
        0.24260404706001282f);
  ffma2(q0, q1, f0, f1, q0, q1, 0.6932762265205383f, 0.6932762265205383f);
  ffma2(q0, q1, f0, f1, q0, q1, 0.9999289512634277f, 0.9999289512634277f);
  p0 = __int_as_float(__float_as_int(q0) + (__float_as_int(r0) << 23));
  p1 = __int_as_float(__float_as_int(q1) + (__float_as_int(r1) << 23));
}

// Pair i (of 32 per 64-key half) takes the FMA-pipe exp2 when kPoly of every
// 32 pairs are to be offloaded (spread evenly, Bresenham).
template <int kPoly>
__device__ __forceinline__ constexpr bool poly_pair(int i) {
  return kPoly > 0 && ((i + 1) * kPoly) / 32 != (i * kPoly) / 32;
}

// bit j set iff base + j < bound (j in [0, 32)).
__device__ __forceinline__ uint32_t lt_bits(int bound, int base) {
  const int n = bound - base;
  return n <= 0 ? 0u : (n >= 32 ? 0xffffffffu : (1u << n) - 1u);
}

__device__ __forceinline__ float exp2_mufu(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <uint32_t kRegs>
__device__ __forceinline__ void reg_alloc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegs));
}
template <uint32_t kRegs>
__device__ __forceinline__ void reg_dealloc() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegs));
}

}  // namespace attn_detail
}  // namespace mrsp
