// Per-event timeline of one tcgen05 decode-attention CTA (dev tool). Builds
// csrc/decode.cu with MRSP_DEC_TRACE and launches one c4-shaped layer (131,109
// prompt keys, 4 KV heads, 7 query heads per KV head, G rows, step t), then
// prints "warp event tile clock" for CTA (0, 0) of the second launch.
//   dec_trace [Lp G streams]
// Events: 0 start, 1 TMA issue (item), 2/3 MMA S(j) wait-K begin/end,
// 4/5/6 MMA P.V(j) wait-P begin / P ready / V ready, 7 softmax S(j) ready,
// 8 softmax P(j) arrived, 9 end.
#define MRSP_DEC_TRACE 1
#include "../../paper_2507_07966_b200/csrc/decode.cu"

#include <cstdio>
#include <cstdlib>
#include <vector>

int main(int argc, char** argv) {
  const int Lp = argc > 1 ? atoi(argv[1]) : 131109;
  const int G = argc > 2 ? atoi(argv[2]) : 8;
  if (argc > 3) setenv("MRSP_DECODE_STREAMS", argv[3], 1);
  const int nq = 28, nkv = 4, qpk = nq / nkv, max_len = 64, t = 0;
  const int kvw = 2 * nkv * 128, Cqkv = (nq + 2 * nkv) * 128;
  std::vector<__nv_bfloat16> h(static_cast<size_t>(2 * nkv) * Lp * 128);
  uint32_t x = 12345;
  for (auto& v : h) {
    x = x * 1664525u + 1013904223u;
    v = __float2bfloat16((static_cast<int>(x >> 9) % 2001 - 1000) * 1e-3f);
  }
  void *prefix, *rows, *q, *part, *out;
  int* tdev;
  cudaMalloc(&prefix, h.size() * 2);
  cudaMemcpy(prefix, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  cudaMalloc(&rows, static_cast<size_t>(max_len) * G * kvw * 2);
  cudaMemset(rows, 0, static_cast<size_t>(max_len) * G * kvw * 2);
  cudaMalloc(&q, static_cast<size_t>(G) * Cqkv * 2);
  cudaMemcpy(q, h.data(), static_cast<size_t>(G) * Cqkv * 2, cudaMemcpyHostToDevice);
  cudaMalloc(&part, mrsp::decode_partial_bytes(Lp, max_len, G, nkv));
  cudaMalloc(&out, static_cast<size_t>(G) * nq * 128 * 2);
  cudaMalloc(&tdev, 4);
  cudaMemcpy(tdev, &t, 4, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 3; ++rep) {
    int zero[12] = {};
    cudaMemcpyToSymbol(mrsp::tc::g_dec_trace_n, zero, sizeof(zero));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    mrsp::decode_attention(q, Cqkv, 0, prefix, rows, kvw, nkv * 128, Lp, G, t, max_len * G, tdev, qpk,
                           nkv, 0.08838834764831845f, static_cast<float*>(part), out, nq * 128, 0);
    cudaEventRecord(b);
    cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    fprintf(stderr, "rep %d: %.1f us (%s)\n", rep, ms * 1e3, cudaGetErrorString(cudaGetLastError()));
  }
  static uint64_t tr[12][mrsp::tc::kDecTraceCap];
  int n[12];
  cudaMemcpyFromSymbol(tr, mrsp::tc::g_dec_trace, sizeof(tr));
  cudaMemcpyFromSymbol(n, mrsp::tc::g_dec_trace_n, sizeof(n));
  for (int w = 0; w < 12; ++w)
    for (int i = 0; i < n[w]; ++i)
      printf("%d %d %d %u\n", w, static_cast<int>(tr[w][i] >> 56),
             static_cast<int>((tr[w][i] >> 32) & 0xffffff), static_cast<uint32_t>(tr[w][i]));
  return 0;
}
