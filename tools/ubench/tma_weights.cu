// Microbenchmark: TMA box-load throughput for the decode GEMMs' weight stream
// (one CTA per SM, `depth` outstanding 16 KB boxes). Each CTA owns a 256-row
// band of a K-major weight [N][K] (the nn.Linear layout) and sweeps K, two
// 128-row boxes per 64-column step (the GEMM's 256 x 64 B tile) — vs the same
// bytes stored band-contiguous (a pre-packed weight: each box 16 KB contiguous).
#include <cstdio>
#include "../../paper_2507_07966_b200/csrc/sm100.cuh"
#include "../../paper_2507_07966_b200/csrc/tma.h"
using namespace mrsp::sm100;

constexpr int BOX_ROWS = 128, BOX_COLS = 64, BOX = BOX_ROWS * BOX_COLS * 2;
__global__ void __launch_bounds__(32, 1) k(const __grid_constant__ CUtensorMap tm, int depth, int n_kb,
                                           int packed, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[16];
  if (threadIdx.x == 0) {
    for (int i = 0; i < depth; ++i) mbar_init(&full[i], 1);
    fence_barrier_init();
  }
  __syncwarp();
  if (threadIdx.x != 0) return;
  const int iters = 2 * n_kb;  // two 128-row boxes per K step
  uint32_t ph[16] = {};
  for (int i = 0; i < iters + depth; ++i) {
    const int s = i % depth;
    if (i >= depth) {
      mbar_wait(&full[s], ph[s]);
      ph[s] ^= 1;
    }
    if (i < iters) {
      mbar_arrive_expect_tx(&full[s], BOX);
      const int kb = i / 2, half = i % 2;
      if (packed)  // band-contiguous: box (band, kb, half) is row block (band * 2 n_kb + 2 kb + half)
        tma_load_2d(smem + s * BOX, &tm, &full[s], 0, ((blockIdx.x * n_kb + kb) * 2 + half) * BOX_ROWS);
      else
        tma_load_2d(smem + s * BOX, &tm, &full[s], kb * BOX_COLS, (blockIdx.x * 2 + half) * BOX_ROWS);
    }
  }
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const long N = 256L * nsm, K = 3584;  // gate/up of the 7B decode step: 37888 x 3584
  const int n_kb = K / BOX_COLS;
  void* buf; cudaMalloc(&buf, N * K * 2);
  cudaMemset(buf, 0, N * K * 2);
  long long* out; cudaMalloc(&out, nsm * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220000);
  CUtensorMap strided = mrsp::make_tmap_bf16_2d(buf, N, K, K, BOX_ROWS, BOX_COLS);
  CUtensorMap packed = mrsp::make_tmap_bf16_2d(buf, N * K / BOX_COLS, BOX_COLS, BOX_COLS, BOX_ROWS, BOX_COLS);
  for (int pk : {0, 1})
    for (int depth : {4, 8, 12}) {
      const CUtensorMap& tm = pk ? packed : strided;
      k<<<nsm, 32, 220000>>>(tm, depth, n_kb, pk, out);
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      for (int r = 0; r < 5; ++r) k<<<nsm, 32, 220000>>>(tm, depth, n_kb, pk, out);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      ms /= 5;
      const double bytes = double(N) * K * 2;
      printf("%-26s depth %2d (%3d KB in flight/SM): %7.0f GB/s, %.1f us per 272 MB (%s)\n",
             pk ? "band-contiguous (packed)" : "K-major [N][K] (strided)", depth, depth * 16,
             bytes / (ms * 1e-3) / 1e9, ms * 1e3, cudaGetErrorString(cudaGetLastError()));
    }
}
