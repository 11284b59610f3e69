// Microbenchmark: MUFU ex2 throughput on sm_100a for f32, f16x2 and bf16x2
// (elements per clock per SM). Used to decide the attention softmax exp path.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

constexpr int ITERS = 4096;
constexpr int CH = 8;

__global__ void k_f32(float* out, float seed, long long* clk) {
  float v[CH];
  for (int i = 0; i < CH; ++i) v[i] = -seed * (threadIdx.x + i) * 1e-3f;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < CH; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}
__global__ void k_bf16x2(float* out, float seed, long long* clk) {
  uint32_t v[CH];
  for (int i = 0; i < CH; ++i) {
    __nv_bfloat162 b = __floats2bfloat162_rn(-seed * (threadIdx.x + i) * 1e-3f, -seed * i * 1e-3f);
    v[i] = *reinterpret_cast<uint32_t*>(&b);
  }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(v[i]));
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < CH; ++i) { __nv_bfloat162 b = *reinterpret_cast<__nv_bfloat162*>(&v[i]); s += __low2float(b) + __high2float(b); }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}
__global__ void k_f16x2(float* out, float seed, long long* clk) {
  uint32_t v[CH];
  for (int i = 0; i < CH; ++i) {
    __half2 b = __floats2half2_rn(-seed * (threadIdx.x + i) * 1e-3f, -seed * i * 1e-3f);
    v[i] = *reinterpret_cast<uint32_t*>(&b);
  }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(v[i]));
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < CH; ++i) { __half2 b = *reinterpret_cast<__half2*>(&v[i]); s += __low2float(b) + __high2float(b); }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float* out; long long* clk; cudaMalloc(&out, 1 << 24); cudaMalloc(&clk, 8);
  const int threads = 512, blocks = nsm;  // 1 block of 16 warps per SM
  auto run = [&](const char* name, void (*k)(float*, float, long long*), int elems_per_op) {
    k<<<blocks, threads>>>(out, 1.f, clk);
    cudaDeviceSynchronize();
    k<<<blocks, threads>>>(out, 1.f, clk);
    cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
    double ops = double(threads) * ITERS * CH;
    printf("%-8s %lld clk  ops/clk/SM %.2f  elems/clk/SM %.2f\n", name, c, ops / c, ops * elems_per_op / c);
  };
  run("f32", k_f32, 1);
  run("bf16x2", k_bf16x2, 2);
  run("f16x2", k_f16x2, 2);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
