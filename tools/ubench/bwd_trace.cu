// Per-phase timeline of one dK / dV CTA of the attention backward (dev tool).
// Builds csrc/backward.cu with MRSP_BWD_TRACE, runs the forward (from the
// library, for a real log-sum-exp) and the backward on a c2-shaped layer, and
// prints per event the clock() stamps of lane 0 of each warp of CTA `cta`.
//   bwd_trace [L Lp Lmax cta kernel]   (kernel 0: dK / dV, 1: dQ)
// Events: TMA warp 20 (ring slot free); MMA warp 10 (stage landed), 11 (S / dP
// issued), 12 (dS of the previous item ready), 13 (its dV / dK issued);
// softmax warps 0 (wait S), 1 (S / dP ready), 2 (loaded), 3 (P / dS computed),
// 4 (stored + arrived).
#define MRSP_BWD_TRACE 1
#include "../../paper_2507_07966_b200/csrc/backward.cu"
#include "../../paper_2507_07966_b200/csrc/attention.h"

#include <cstdio>
#include <vector>

int main(int argc, char** argv) {
  const int L = argc > 1 ? atoi(argv[1]) : 16421 + 8 * 1024;
  const int Lp = argc > 2 ? atoi(argv[2]) : 16421;
  const int Lmax = argc > 3 ? atoi(argv[3]) : 1024;
  const int cta = argc > 4 ? atoi(argv[4]) : 8;
  const int kernel = argc > 5 ? atoi(argv[5]) : 0;  // 0: dK / dV, 1: dQ
  const int nq = 28, nkv = 4, C = (nq + 2 * nkv) * 128, Cq = nq * 128;
  std::vector<__nv_bfloat16> h(static_cast<size_t>(L) * C), hd(static_cast<size_t>(L) * Cq);
  uint32_t x = 12345;
  for (auto& v : h) {
    x = x * 1664525u + 1013904223u;
    v = __float2bfloat16((static_cast<int>(x >> 9) % 2001 - 1000) * 2e-3f);
  }
  for (auto& v : hd) {
    x = x * 1664525u + 1013904223u;
    v = __float2bfloat16((static_cast<int>(x >> 9) % 2001 - 1000) * 1e-3f);
  }
  void *qkv, *o, *dO, *dqkv;
  float *lse, *D;
  const int ld = (L + 3) / 4 * 4;
  cudaMalloc(&qkv, h.size() * 2);
  cudaMalloc(&o, hd.size() * 2);
  cudaMalloc(&dO, hd.size() * 2);
  cudaMalloc(&dqkv, h.size() * 2);
  cudaMalloc(&lse, static_cast<size_t>(nq) * ld * 4);
  cudaMalloc(&D, static_cast<size_t>(nq) * ld * 4);
  cudaMemcpy(qkv, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dO, hd.data(), hd.size() * 2, cudaMemcpyHostToDevice);
  mrsp::AttnParams fp{qkv, C, 0, qkv, C, nq * 128, qkv, C, (nq + nkv) * 128, o, Cq, 0,
                      L, nq, nq / nkv, 0.08838834764831845f, ATTN_CAUSAL_PREFIX, Lp, Lmax, 0};
  fp.lse = lse;
  fp.lse_ld = ld;
  mrsp::attention_fwd(fp, 0);
  cudaMemcpyToSymbol(mrsp::g_bwd_trace_cta, &cta, sizeof(int));
  cudaMemcpyToSymbol(mrsp::g_bwd_trace_kernel, &kernel, sizeof(int));
  mrsp::AttnBwdParams bp{qkv, C, 0, nq * 128, (nq + nkv) * 128, o, Cq, dO, Cq, lse, D, ld, dqkv, C,
                         L, nq, nq / nkv, 0.08838834764831845f, Lp, Lmax};
  for (int rep = 0; rep < 3; ++rep) {
    int zero[12] = {};
    cudaMemcpyToSymbol(mrsp::g_bwd_trace_n, zero, sizeof(zero));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    mrsp::attention_bwd(bp, 0);
    cudaEventRecord(b);
    cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    fprintf(stderr, "rep %d: dq + dkdv %.3f ms (%s)\n", rep, ms, cudaGetErrorString(cudaGetLastError()));
  }
  static uint64_t tr[12][mrsp::kBTraceCap];
  int n[12];
  cudaMemcpyFromSymbol(tr, mrsp::g_bwd_trace, sizeof(tr));
  cudaMemcpyFromSymbol(n, mrsp::g_bwd_trace_n, sizeof(n));
  for (int w = 0; w < 12; ++w)
    for (int i = 0; i < n[w]; ++i)
      printf("%d %d %d %u\n", w, static_cast<int>(tr[w][i] >> 56),
             static_cast<int>((tr[w][i] >> 32) & 0xffffff), static_cast<uint32_t>(tr[w][i]));
  return 0;
}
