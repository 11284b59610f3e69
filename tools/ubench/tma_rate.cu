// Microbenchmark: TMA 2-D box-load throughput per SM (one CTA per SM, a ring
// of `depth` outstanding 16 KB boxes), for the attention K/V access pattern:
// rows of 128 B (64 bf16) at a pitch of `pitch` elements, each CTA sweeping
// its own or a shared row range. Reports aggregate GB/s.
#include <cstdio>
#include <vector>
#include "../../paper_2507_07966_b200/csrc/sm100.cuh"
#include "../../paper_2507_07966_b200/csrc/tma.h"
using namespace mrsp::sm100;

constexpr int BOX_ROWS = 128, BOX_COLS = 64, BOX = BOX_ROWS * BOX_COLS * 2;
__global__ void __launch_bounds__(32, 1) k(const __grid_constant__ CUtensorMap tm, int depth, int iters,
                                           int rows, int ncolblk, int shared_sweep, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[16];
  if (threadIdx.x == 0) {
    for (int i = 0; i < depth; ++i) mbar_init(&full[i], 1);
    fence_barrier_init();
  }
  __syncwarp();
  if (threadIdx.x != 0) return;
  const int nrb = rows / BOX_ROWS;
  // CTAs start at different row blocks unless shared_sweep (all sweep together)
  int rb = shared_sweep ? 0 : (blockIdx.x * 37) % nrb;
  const int cb = blockIdx.x % ncolblk;
  long long t0 = clock64();
  uint32_t ph[16] = {};
  for (int i = 0; i < iters + depth; ++i) {
    const int s = i % depth;
    if (i >= depth) {  // wait for the load issued depth iterations ago
      mbar_wait(&full[s], ph[s]);
      ph[s] ^= 1;
    }
    if (i < iters) {
      mbar_arrive_expect_tx(&full[s], BOX);
      tma_load_2d(smem + s * BOX, &tm, &full[s], cb * BOX_COLS, rb * BOX_ROWS);
      if (++rb == nrb) rb = 0;
    }
  }
  long long t1 = clock64();
  out[blockIdx.x] = t1 - t0;
}


// 2-CTA variant: cluster of 2; both CTAs load their own box into own smem and
// complete the bytes on the LEADER's barrier (cp.async.bulk.tensor.cta_group::2);
// the leader waits, then frees the slot in both CTAs with a remote arrive.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(32, 1)
    k2(const __grid_constant__ CUtensorMap tm, int depth, int iters, int rows, int ncolblk, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[16], empty[16];
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    for (int i = 0; i < depth; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    fence_barrier_init();
  }
  cluster_sync();
  if (threadIdx.x == 0) {
    const int nrb = rows / BOX_ROWS;
    int rb = 0;
    const int cb = (blockIdx.x >> 1) % ncolblk;
    long long t0 = clock64();
    uint32_t ph[16] = {}, eph[16] = {};
    for (int i = 0; i < iters + depth; ++i) {
      const int s = i % depth;
      if (i >= depth) {
        if (rank == 0) {  // leader: both halves landed -> free the slot in both CTAs
          mbar_wait(&full[s], ph[s]);
          ph[s] ^= 1;
          mbar_arrive(&empty[s]);
          mbar_arrive_remote(mapa_shared(smem_u32(&empty[s]), 1));
        }
      }
      if (i < iters) {
        if (i >= depth) { mbar_wait(&empty[s], eph[s]); eph[s] ^= 1; }
        if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * BOX);
        tma_load_2d_2sm(smem + s * BOX, &tm, &full[s], cb * BOX_COLS + rank * 0, (rb * 2 + rank) * BOX_ROWS % rows);
        if (++rb == nrb / 2) rb = 0;
      }
    }
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  cluster_sync();
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int clk_khz; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const long rows = 139264;
  long long* out; cudaMalloc(&out, nsm * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  struct Cfg { const char* name; long cols; int ncolblk; };
  // qkv layout: 36 heads x 128 cols per token row; K/V of 4 kv heads = 8 col blocks of 64
  // contiguous: a [head][L][128] tensor -> pitch 128 cols
  for (Cfg c : {Cfg{"qkv pitch 4608 (K/V strided)", 4608, 16}, Cfg{"per-head pitch 128 (contiguous)", 128, 2}}) {
    void* buf; cudaMalloc(&buf, rows * c.cols * 2);
    cudaMemset(buf, 0, rows * c.cols * 2);
    CUtensorMap tm = mrsp::make_tmap_bf16_2d(buf, rows, c.cols, c.cols, BOX_ROWS, BOX_COLS);
    for (int shared_sweep : {0, 1})
      for (int depth : {2, 4, 8, 12}) {
        const int iters = 2000;
        k<<<nsm, 32, 200000>>>(tm, depth, iters, rows, c.ncolblk, shared_sweep, out);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        k<<<nsm, 32, 200000>>>(tm, depth, iters, rows, c.ncolblk, shared_sweep, out);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double gbs = double(nsm) * iters * BOX / (ms * 1e-3) / 1e9;
        printf("%-34s sweep=%s depth %2d: %7.0f GB/s aggregate, %5.1f GB/s/SM, %.2f us per box per SM (%s)\n",
               c.name, shared_sweep ? "shared" : "spread", depth, gbs, gbs / nsm,
               ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
      }
    for (int depth : {4, 8, 12}) {
      const int iters = 2000;
      cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
      k2<<<nsm, 32, 200000>>>(tm, depth, iters, rows, c.ncolblk, out);
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      k2<<<nsm, 32, 200000>>>(tm, depth, iters, rows, c.ncolblk, out);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double gbs = double(nsm) * iters * BOX / (ms * 1e-3) / 1e9;
      printf("%-34s 2SM-TMA pair sweep depth %2d: %7.0f GB/s aggregate, %5.1f GB/s/SM (%s)\n", c.name, depth,
             gbs, gbs / nsm, cudaGetErrorString(cudaGetLastError()));
    }
    cudaFree(buf);
  }
}
