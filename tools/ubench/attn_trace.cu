// Per-phase timeline of one attention CTA (dev tool). Builds csrc/attention.cu
// with MRSP_ATTN_TRACE and prints, per event, the clock() stamps of lane 0 of
// each warp for the CTA `cta` of a c4-shaped (or given) launch.
//   attn_trace [L Lp Lmax cta]
#define MRSP_ATTN_TRACE 1
#ifdef GLOBAL_CLOCK
#define MRSP_ATTN_TRACE_GLOBAL 1
#endif
#include "../../paper_2507_07966_b200/csrc/attention.cu"

#include <cstdio>
#include <vector>

int main(int argc, char** argv) {
  const int L = argc > 1 ? atoi(argv[1]) : 139197;
  const int Lp = argc > 2 ? atoi(argv[2]) : 131109;
  const int Lmax = argc > 3 ? atoi(argv[3]) : 1011;
  const int cta = argc > 4 ? atoi(argv[4]) : 0;
  const int nq = 28, nkv = 4, C = (nq + 2 * nkv) * 128;
  std::vector<__nv_bfloat16> h(static_cast<size_t>(L) * C);
  uint32_t x = 12345;
  for (auto& v : h) {
    x = x * 1664525u + 1013904223u;
    v = __float2bfloat16((static_cast<int>(x >> 9) % 2001 - 1000) * 1e-3f);
  }
  void *qkv, *o;
  cudaMalloc(&qkv, h.size() * 2);
  cudaMalloc(&o, static_cast<size_t>(L) * nq * 128 * 2);
  cudaMemcpy(qkv, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpyToSymbol(mrsp::g_attn_trace_cta, &cta, sizeof(int));
  mrsp::AttnParams p{qkv, C, 0, qkv, C, nq * 128, qkv, C, (nq + nkv) * 128, o, nq * 128, 0,
                     L, nq, nq / nkv, 0.08838834764831845f, ATTN_CAUSAL_PREFIX, Lp, Lmax, 0};
  for (int rep = 0; rep < 2; ++rep) {
    int zero[24] = {};
    cudaMemcpyToSymbol(mrsp::g_attn_trace_n, zero, sizeof(zero));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    mrsp::attention_fwd(p, 0);
    cudaEventRecord(b);
    cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    fprintf(stderr, "rep %d: %.3f ms (%s)\n", rep, ms, cudaGetErrorString(cudaGetLastError()));
  }
  static uint64_t tr[24][mrsp::kTraceCap];
  int n[24];
  cudaMemcpyFromSymbol(tr, mrsp::g_attn_trace, sizeof(tr));
  cudaMemcpyFromSymbol(n, mrsp::g_attn_trace_n, sizeof(n));
  for (int w = 0; w < 24; ++w)
    for (int i = 0; i < n[w]; ++i)
      printf("%d %d %d %u\n", w, static_cast<int>(tr[w][i] >> 56),
             static_cast<int>((tr[w][i] >> 32) & 0xffffff), static_cast<uint32_t>(tr[w][i]));
  return 0;
}
