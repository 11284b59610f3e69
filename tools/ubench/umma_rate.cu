// Microbenchmark: tcgen05.mma kind::f16 throughput (FLOP/clk/SM) for
// M=128 x N x K=16 with A from smem (ss) or TMEM (ts), B from smem.
// Operand contents are irrelevant (uninitialised smem).
#include <cstdio>
#include "../../paper_2507_07966_b200/csrc/sm100.cuh"
using namespace mrsp::sm100;

constexpr int REPS = 2048;
template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) k(long long* clk) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&slot);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 1) {
    const uint32_t idesc = TS ? idesc_bf16_f32_bmn(128, N) : idesc_bf16_f32(128, N);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 65536);
    long long t0 = clock64();
    if (elect_one()) {
      for (int r = 0; r < REPS; ++r)
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          if (TS)
            mma_bf16_ts(tmem + 256, tmem + kk * 8, sdesc_sw128_mn(b + kk * 2048, 16384), idesc, 1u);
          else
            mma_bf16_ss(tmem + 256, sdesc_sw128(a + (kk / 4) * 16384 + (kk % 4) * 32),
                        sdesc_sw128(b + (kk / 4) * 16384 + (kk % 4) * 32), idesc, 1u);
        }
      mma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 32 && blockIdx.x == 0) *clk = t1 - t0;
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int N, bool TS>
void run(long long* d) {
  cudaFuncSetAttribute(k<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  k<N, TS><<<nsm, 128, 140000>>>(d);
  k<N, TS><<<nsm, 128, 140000>>>(d);
  cudaDeviceSynchronize();
  long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  double flop = 2.0 * 128 * N * 16 * 8 * REPS;
  printf("M128 N%3d %s: %lld clk  %.0f flop/clk/SM  (%.1f%% of 8192)  smem B/clk %.1f  err=%s\n", N,
         TS ? "ts" : "ss", c, flop / c, 100 * flop / c / 8192,
         (TS ? 0.0 : 128.0 * 16 * 2) * 8 * REPS / c + (N * 16 * 2.0) * 8 * REPS / c,
         cudaGetErrorString(cudaGetLastError()));
}

// CTA-pair variant: cluster of 2, leader issues tcgen05.mma.cta_group::2 (M=256).
template <int N, bool TS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k2(long long* clk) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  const bool leader = cluster_ctarank() == 0;
  if (warp == 0) tmem_alloc_pair<512>(&slot);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  tc_fence_before(); cluster_sync(); tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 1) {
    const uint32_t idesc = TS ? idesc_bf16_f32_bmn(256, N) : idesc_bf16_f32(256, N);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 65536);
    long long t0 = clock64();
    if (leader && elect_one()) {
      for (int r = 0; r < REPS; ++r)
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          if (TS)
            mma2_bf16_ts(tmem + 256, tmem + kk * 8, sdesc_sw128_mn(b + kk * 2048, 16384), idesc, 1u);
          else
            mma2_bf16_ss(tmem + 256, sdesc_sw128(a + (kk / 4) * 16384 + (kk % 4) * 32),
                         sdesc_sw128(b + (kk / 4) * 8192 + (kk % 4) * 32), idesc, 1u);
        }
      mma_commit_pair(&bar, 3);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 32 && blockIdx.x == 0) *clk = t1 - t0;
  }
  tc_fence_before(); cluster_sync(); tc_fence_after();
  if (warp == 0) tmem_dealloc_pair<512>(tmem);
}
template <int N, bool TS>
void run2(long long* d) {
  cudaFuncSetAttribute(k2<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  k2<N, TS><<<nsm, 128, 140000>>>(d);
  k2<N, TS><<<nsm, 128, 140000>>>(d);
  cudaDeviceSynchronize();
  long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  double flop_per_sm = 2.0 * 128 * N * 16 * 8 * REPS;  // each SM computes 128 of the 256 rows
  printf("PAIR M256 N%3d %s: %lld clk  %.0f flop/clk/SM  (%.1f%% of 8192)  err=%s\n", N, TS ? "ts" : "ss", c,
         flop_per_sm / c, 100 * flop_per_sm / c / 8192, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* d; cudaMalloc(&d, 8);
  run<64, false>(d); run<128, false>(d); run<256, false>(d);
  run<64, true>(d); run<128, true>(d); run<256, true>(d);
  run2<128, false>(d); run2<256, false>(d); run2<128, true>(d); run2<256, true>(d);
}
