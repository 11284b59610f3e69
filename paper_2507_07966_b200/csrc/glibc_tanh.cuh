// glibc_tanh.cuh — fp64 tanh on the device, bit-identical to the host libm the
// reference links (glibc 2.39, x86_64, FMA ifunc variant of expm1).
//
// Why: the reference's tests compare the engine path to the serial CPU path
// with operator== on doubles (test_grpo.cpp:344-369, acceptance.cpp:345-404),
// and policy.cpp:47/:97 call std::tanh. CUDA's tanh differs from glibc's in
// ~0.1% of inputs by 1 ulp, so the toy path evaluates glibc's algorithm
// (fdlibm s_tanh.c over s_expm1.c, with the Estrin polynomial and the FMA
// sites GCC emits for the -mfma multiarch build) using explicitly rounded
// intrinsics — nvcc may not contract anything here. Verified identical to
// glibc on 4e7 random inputs (tests/test_oracle.py::test_glibc_tanh_model).
#pragma once

namespace mrsp {

__device__ __forceinline__ unsigned hi_word(double x) {
  return static_cast<unsigned>(__double_as_longlong(x) >> 32);
}
__device__ __forceinline__ double with_hi_word(double x, unsigned h) {
  long long u = __double_as_longlong(x);
  u = (u & 0xffffffffLL) | (static_cast<long long>(h) << 32);
  return __longlong_as_double(u);
}

#define DADD(a, b) __dadd_rn((a), (b))
#define DSUB(a, b) __dadd_rn((a), -(b))
#define DMUL(a, b) __dmul_rn((a), (b))
#define DDIV(a, b) __ddiv_rn((a), (b))
#define DFMA(a, b, c) __fma_rn((a), (b), (c))

__device__ inline double glibc_expm1(double x) {
  const double one = 1.0, tiny = 1.0e-300;
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10,
               invln2 = 1.44269504088896338700e+00;
  const double Q1 = -3.33333333333331316428e-02, Q2 = 1.58730158725481460165e-03,
               Q3 = -7.93650757867487942473e-05, Q4 = 4.00821782732936239552e-06,
               Q5 = -2.01099218183624371326e-07;
  double y, hi, lo, c = 0.0, t, e, hxs, hfx, r1;
  int k;
  unsigned hx = hi_word(x);
  const unsigned xsb = hx & 0x80000000u;
  hx &= 0x7fffffffu;
  if (hx >= 0x4043687Au && xsb) return DSUB(tiny, one);  // x < -56 ln2
  if (hx > 0x3fd62e42u) {
    if (hx < 0x3FF0A2B2u) {
      if (!xsb) { hi = DSUB(x, ln2_hi); lo = ln2_lo; k = 1; }
      else { hi = DADD(x, ln2_hi); lo = -ln2_lo; k = -1; }
    } else {
      k = static_cast<int>(DFMA(invln2, x, xsb == 0 ? 0.5 : -0.5));
      t = static_cast<double>(k);
      hi = DFMA(-t, ln2_hi, x);
      lo = DMUL(t, ln2_lo);
    }
    x = DSUB(hi, lo);
    c = DSUB(DSUB(hi, x), lo);
  } else if (hx < 0x3c900000u) {
    return x;
  } else {
    k = 0;
  }
  hfx = DMUL(0.5, x);
  hxs = DMUL(x, hfx);
  const double R1 = DFMA(hxs, Q1, one), h2 = DMUL(hxs, hxs), R2 = DFMA(hxs, Q3, Q2),
               h4 = DMUL(h2, h2), R3 = DFMA(hxs, Q5, Q4);
  r1 = DFMA(h4, R3, DFMA(h2, R2, R1));
  t = DFMA(-r1, hfx, 3.0);
  e = DMUL(hxs, DDIV(DSUB(r1, t), DFMA(-x, t, 6.0)));
  if (k == 0) return DSUB(x, DFMA(x, e, -hxs));
  e = DFMA(x, DSUB(e, c), -c);
  e = DSUB(e, hxs);
  if (k == -1) return DFMA(0.5, DSUB(x, e), -0.5);
  if (k == 1) {
    if (x < -0.25) return DMUL(-2.0, DSUB(e, DADD(x, 0.5)));
    return DFMA(2.0, DSUB(x, e), one);
  }
  if (k <= -2 || k > 56) {
    y = DSUB(one, DSUB(e, x));
    y = with_hi_word(y, hi_word(y) + (static_cast<unsigned>(k) << 20));
    return DSUB(y, one);
  }
  if (k < 20) {
    t = with_hi_word(one, 0x3ff00000u - (0x200000u >> k));
    y = DSUB(t, DSUB(e, x));
    y = with_hi_word(y, hi_word(y) + (static_cast<unsigned>(k) << 20));
  } else {
    t = with_hi_word(0.0, static_cast<unsigned>(0x3ff - k) << 20);
    y = DSUB(x, DADD(e, t));
    y = DADD(y, one);
    y = with_hi_word(y, hi_word(y) + (static_cast<unsigned>(k) << 20));
  }
  return y;
}

__device__ inline double glibc_tanh(double x) {
  const unsigned jx = hi_word(x), ix = jx & 0x7fffffffu;
  double t, z;
  if (ix >= 0x7ff00000u) return x != x ? x : (static_cast<int>(jx) >= 0 ? 1.0 : -1.0);
  if (ix < 0x40360000u) {  // |x| < 22
    if (ix < 0x3c800000u) return DMUL(x, DADD(1.0, x));
    if (ix >= 0x3ff00000u) {
      t = glibc_expm1(DMUL(2.0, fabs(x)));
      z = DSUB(1.0, DDIV(2.0, DADD(t, 2.0)));
    } else {
      t = glibc_expm1(DMUL(-2.0, fabs(x)));
      z = DDIV(-t, DADD(t, 2.0));
    }
  } else {
    z = DSUB(1.0, 1.0e-300);
  }
  return static_cast<int>(jx) >= 0 ? z : -z;
}

}  // namespace mrsp
