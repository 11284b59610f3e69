// rownorm.cuh — RMSNorm of one row by a whole CTA, for the decode fusions
// (split-K residual reduction + norm, token embedding + norm).
//
// Bit-identical to rmsnorm_kernel (csrc/kernels_misc.cu): warp 0 forms the
// sum of squares in that kernel's order (lane-strided float4 chunks, then the
// xor butterfly), and every output element is bf16(w * (x * r)).
#pragma once

#include <cuda_bf16.h>

namespace mrsp {

__device__ __forceinline__ float rownorm_warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// x: the row (fp32, 16-byte aligned, written by this CTA before the call and
// made visible with __syncthreads()); d % 4 == 0. All threads of the CTA call.
__device__ __forceinline__ void block_rmsnorm_row(const float* x, const float* __restrict__ w,
                                                  __nv_bfloat16* __restrict__ out, int d,
                                                  float eps) {
  __shared__ float s_r;
  const float4* xr = reinterpret_cast<const float4*>(x);
  if (threadIdx.x < 32) {
    float ss = 0.f;
    for (int i = threadIdx.x; i < d / 4; i += 32) {
      const float4 v = xr[i];
      ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    }
    ss = rownorm_warp_sum(ss);
    if (threadIdx.x == 0) s_r = rsqrtf(ss / static_cast<float>(d) + eps);
  }
  __syncthreads();
  const float r = s_r;
  const float4* wr = reinterpret_cast<const float4*>(w);
  __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>(out);
  for (int i = threadIdx.x; i < d / 4; i += blockDim.x) {
    const float4 v = xr[i], g = wr[i];
    o[2 * i] = __floats2bfloat162_rn(g.x * (v.x * r), g.y * (v.y * r));
    o[2 * i + 1] = __floats2bfloat162_rn(g.z * (v.z * r), g.w * (v.w * r));
  }
}

}  // namespace mrsp
