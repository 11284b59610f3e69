// Does the bf16x2 pack (cvt.rn.bf16x2.f32 -> F2FP) share the MUFU (XU) pipe
// with ex2.approx? (dev tool) Each kernel runs `iters` rounds of 8 independent
// chains per thread; prints clocks per warp-instruction per SM sub-partition.
#include <cstdint>
#include <cstdio>
#include <cuda_bf16.h>

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack(float a, float b) {
  uint32_t r;
  asm volatile("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(r) : "f"(a), "f"(b));
  return r;
}

template <int kMode>  // 0: ex2 only, 1: pack only, 2: ex2 + pack (2 ex2 per pack), 3: int RNE pack
__global__ void k(float* out, int iters, long long* clk) {
  float x[8];
  uint32_t acc = 0;
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      if (kMode == 0 || kMode == 2) {
        x[i] = ex2(x[i]) * -0.5f;
        x[i + 1] = ex2(x[i + 1]) * -0.5f;
      }
      if (kMode == 1 || kMode == 2) {
        acc ^= pack(x[i], x[i + 1]);
        x[i] += 1e-7f;
      }
      if (kMode == 3) {
        uint32_t u0 = __float_as_uint(x[i]), u1 = __float_as_uint(x[i + 1]);
        u0 = u0 + 0x7fffu + ((u0 >> 16) & 1u);
        u1 = u1 + 0x7fffu + ((u1 >> 16) & 1u);
        acc ^= __byte_perm(u0, u1, 0x7632);
        x[i] += 1e-7f;
      }
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

template <int kMode>
void run(const char* name, int warps) {
  float* out;
  long long* clk;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&clk, 8);
  const int iters = 4096;
  k<kMode><<<148, warps * 32>>>(out, iters, clk);
  k<kMode><<<148, warps * 32>>>(out, iters, clk);
  long long c;
  cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
  // warp-instructions of the measured kind per SMSP: warps/4 * iters * 4 pairs
  const double per_smsp = (warps / 4.0) * iters * 4;
  printf("%-28s warps/SM %2d: %8lld clk, %.2f clk per pair-round per SMSP\n", name, warps, c, c / per_smsp);
  cudaFree(out);
  cudaFree(clk);
}

int main() {
  for (int w : {4, 8, 16}) {
    run<0>("ex2 x2", w);
    run<1>("cvt.rn.bf16x2 x1", w);
    run<2>("ex2 x2 + cvt x1", w);
    run<3>("int RNE pack x1", w);
  }
  return 0;
}
