// toy.cu — the reference's own MR-SP model on the device, fp64, bit-exact.
//
// Kernels
//   toy_encode_kernel   encode_frame (policy.cpp:36-47) for a rank's frame range:
//                       e[f][r] = tanh(sum_k W[r][k] * x[f][k]), k ascending,
//                       each product and sum individually rounded (no FMA),
//                       tanh = glibc_tanh. One CTA per frame, one thread per r.
//   toy_prefill_kernel  step_logits (policy.cpp:85-119) for a rank's positions:
//                       s = tanh(c + sum_k (A[r][k] ctx[k] + B[r][k] E[prev][k]))
//                       logits[v] = b[v] + sum_r U[v][r] s[r].
// Both reproduce the reference's summation order exactly, so the device
// result equals the reference CPU bit for bit (tests/test_toy_gpu.py).
// Ranks are CUDA streams on the current device; each launches only its own
// ShardPlan range (engine.cpp:85-100, :117-129).
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "common.h"
#include "glibc_tanh.cuh"

namespace mrsp {
namespace {

__global__ void toy_encode_kernel(const double* __restrict__ w, const double* __restrict__ frames,
                                  double* __restrict__ out, int d, int p, uint64_t f_begin) {
  extern __shared__ double xs[];  // one frame
  const uint64_t f = f_begin + blockIdx.x;
  const double* x = frames + f * static_cast<uint64_t>(p);
  for (int k = threadIdx.x; k < p; k += blockDim.x) xs[k] = x[k];
  __syncthreads();
  for (int r = threadIdx.x; r < d; r += blockDim.x) {
    const double* row = w + static_cast<uint64_t>(r) * p;
    double z = 0.0;
    for (int k = 0; k < p; ++k) z = DADD(z, DMUL(row[k], xs[k]));
    out[f * static_cast<uint64_t>(d) + r] = glibc_tanh(z);
  }
}

struct Pos {
  uint32_t row;
  int32_t prev;
  uint64_t out_index;
};

__global__ void toy_prefill_kernel(const double* __restrict__ theta, const double* __restrict__ ctxs,
                                   const Pos* __restrict__ pos, double* __restrict__ out, int V,
                                   int d, int h) {
  extern __shared__ double sm[];
  double* ctx = sm;          // d
  double* e_prev = sm + d;   // d
  double* s = sm + 2 * d;    // h
  const Pos ps = pos[blockIdx.x];
  const double* E = theta;
  const double* A = theta + static_cast<uint64_t>(V) * d;
  const double* B = A + static_cast<uint64_t>(h) * d;
  const double* c = B + static_cast<uint64_t>(h) * d;
  const double* U = c + h;
  const double* bias = U + static_cast<uint64_t>(V) * h;
  for (int k = threadIdx.x; k < d; k += blockDim.x) {
    ctx[k] = ctxs[static_cast<uint64_t>(ps.row) * d + k];
    e_prev[k] = E[static_cast<uint64_t>(ps.prev) * d + k];
  }
  __syncthreads();
  for (int r = threadIdx.x; r < h; r += blockDim.x) {
    const double* arow = A + static_cast<uint64_t>(r) * d;
    const double* brow = B + static_cast<uint64_t>(r) * d;
    double z = c[r];
    for (int k = 0; k < d; ++k) z = DADD(z, DADD(DMUL(arow[k], ctx[k]), DMUL(brow[k], e_prev[k])));
    s[r] = glibc_tanh(z);
  }
  __syncthreads();
  for (int v = threadIdx.x; v < V; v += blockDim.x) {
    const double* urow = U + static_cast<uint64_t>(v) * h;
    double z = bias[v];
    for (int r = 0; r < h; ++r) z = DADD(z, DMUL(urow[r], s[r]));
    out[ps.out_index * static_cast<uint64_t>(V) + v] = z;
  }
}

// Per-process pool of rank streams (ranks = streams on the current device).
std::vector<cudaStream_t>& rank_streams(int k) {
  static std::mutex mu;
  static std::vector<cudaStream_t> pool;
  std::lock_guard<std::mutex> lock(mu);
  while (static_cast<int>(pool.size()) < k) {
    cudaStream_t s;
    MRSP_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    pool.push_back(s);
  }
  return pool;
}

template <typename T>
struct DevBuf {
  T* p = nullptr;
  explicit DevBuf(size_t n) {
    if (n) MRSP_CUDA(cudaMalloc(&p, n * sizeof(T)));
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

void check_plan(const uint64_t* ranges, int k, uint64_t total, const char* who) {
  uint64_t cursor = 0;
  for (int w = 0; w < k; ++w) {
    MRSP_REQUIRE(ranges[2 * w] <= ranges[2 * w + 1] && ranges[2 * w + 1] <= total,
                 MRSP_INVALID_ARGUMENT, std::string(who) + ": malformed plan range");
    MRSP_REQUIRE(ranges[2 * w] == cursor, MRSP_INVALID_ARGUMENT,
                 std::string(who) + ": plan ranges are not a contiguous partition");
    cursor = ranges[2 * w + 1];
  }
  MRSP_REQUIRE(cursor == total, MRSP_INVALID_ARGUMENT,
               std::string(who) + ": plan does not cover its items");
}

}  // namespace
}  // namespace mrsp

using namespace mrsp;

extern "C" mrsp_status mrsp_toy_encode(int sp_degree, const double* enc_w, int d, int p,
                                       const double* frames, uint64_t n_frames,
                                       const uint64_t* ranges, double* out,
                                       uint64_t* rank_items) {
  return guard([&] {
    MRSP_REQUIRE(sp_degree >= 1, MRSP_INVALID_ARGUMENT, "WorkerGroup: sp_degree must be >= 1");
    MRSP_REQUIRE(d >= 1 && p >= 1, MRSP_INVALID_ARGUMENT, "encode_frame: frame dimension mismatch");
    check_plan(ranges, sp_degree, n_frames, "parallel_encode");
    require_device();
    if (n_frames == 0) {
      for (int w = 0; w < sp_degree; ++w) rank_items[w] = 0;
      return;
    }
    auto& streams = rank_streams(sp_degree);
    DevBuf<double> dw(static_cast<size_t>(d) * p), dx(n_frames * p), dout(n_frames * d);
    MRSP_CUDA(cudaMemcpyAsync(dw.p, enc_w, sizeof(double) * d * p, cudaMemcpyHostToDevice, streams[0]));
    MRSP_CUDA(cudaMemcpyAsync(dx.p, frames, sizeof(double) * n_frames * p, cudaMemcpyHostToDevice,
                              streams[0]));
    cudaEvent_t ready;
    MRSP_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    MRSP_CUDA(cudaEventRecord(ready, streams[0]));
    const int threads = std::min(256, ((d + 31) / 32) * 32);
    for (int w = 0; w < sp_degree; ++w) {
      const uint64_t b = ranges[2 * w], e = ranges[2 * w + 1];
      rank_items[w] = e - b;
      if (e == b) continue;
      MRSP_CUDA(cudaStreamWaitEvent(streams[w], ready, 0));
      toy_encode_kernel<<<static_cast<unsigned>(e - b), threads, sizeof(double) * p, streams[w]>>>(
          dw.p, dx.p, dout.p, d, p, b);
      count_launch();
      MRSP_CUDA(cudaGetLastError());
      // each rank's slice lands in its own range of the gathered buffer
      MRSP_CUDA(cudaMemcpyAsync(out + b * d, dout.p + b * d, sizeof(double) * (e - b) * d,
                                cudaMemcpyDeviceToHost, streams[w]));
    }
    for (int w = 0; w < sp_degree; ++w) MRSP_CUDA(cudaStreamSynchronize(streams[w]));
    cudaEventDestroy(ready);
  });
}

extern "C" mrsp_status mrsp_toy_prefill(int sp_degree, const double* theta, int V, int d, int h,
                                        const double* contexts, const int32_t* rows,
                                        const uint64_t* lengths, uint64_t n_rows,
                                        uint64_t max_len, const uint64_t* ranges, double* out,
                                        uint64_t* pad_reads) {
  return guard([&] {
    MRSP_REQUIRE(sp_degree >= 1, MRSP_INVALID_ARGUMENT, "WorkerGroup: sp_degree must be >= 1");
    MRSP_REQUIRE(V >= 1 && d >= 1 && h >= 1, MRSP_INVALID_ARGUMENT, "prefill: bad policy dims");
    check_plan(ranges, sp_degree, max_len, "parallel_prefill");
    require_device();
    *pad_reads = 0;
    // Output offsets of each row in the packed [sum(len)][V] result.
    std::vector<uint64_t> row_off(n_rows + 1, 0);
    for (uint64_t r = 0; r < n_rows; ++r) {
      MRSP_REQUIRE(lengths[r] <= max_len, MRSP_INVALID_ARGUMENT, "prefill: row longer than max_len");
      row_off[r + 1] = row_off[r] + lengths[r];
    }
    const uint64_t total = row_off[n_rows];
    if (total == 0) return;
    // Each rank's position list: t in [b, min(e, len_r)) for every row
    // (engine.cpp:120-123); prev is read only below len_r, so no pad reads.
    std::vector<std::vector<Pos>> plist(sp_degree);
    for (int w = 0; w < sp_degree; ++w) {
      const uint64_t b = ranges[2 * w], e = ranges[2 * w + 1];
      for (uint64_t r = 0; r < n_rows; ++r) {
        const uint64_t stop = std::min(e, static_cast<uint64_t>(lengths[r]));
        for (uint64_t t = b; t < stop; ++t) {
          int32_t prev = 1;  // Vocab::kEos
          if (t > 0) {
            if (t - 1 >= lengths[r]) ++*pad_reads;
            prev = rows[r * max_len + t - 1];
          }
          MRSP_REQUIRE(prev >= 0 && prev < V, MRSP_INVALID_ARGUMENT,
                       "step_logits: prev token out of range");
          plist[w].push_back(Pos{static_cast<uint32_t>(r), prev, row_off[r] + t});
        }
      }
    }
    const uint64_t n_theta = static_cast<uint64_t>(V) * d + 2ull * h * d + h +
                             static_cast<uint64_t>(V) * h + V;
    auto& streams = rank_streams(sp_degree);
    DevBuf<double> dtheta(n_theta), dctx(n_rows * d), dout(total * V);
    DevBuf<Pos> dpos(total);
    MRSP_CUDA(cudaMemcpyAsync(dtheta.p, theta, sizeof(double) * n_theta, cudaMemcpyHostToDevice,
                              streams[0]));
    MRSP_CUDA(cudaMemcpyAsync(dctx.p, contexts, sizeof(double) * n_rows * d, cudaMemcpyHostToDevice,
                              streams[0]));
    uint64_t off = 0;
    std::vector<uint64_t> pos_off(sp_degree);
    for (int w = 0; w < sp_degree; ++w) {
      pos_off[w] = off;
      if (!plist[w].empty())
        MRSP_CUDA(cudaMemcpyAsync(dpos.p + off, plist[w].data(), sizeof(Pos) * plist[w].size(),
                                  cudaMemcpyHostToDevice, streams[0]));
      off += plist[w].size();
    }
    cudaEvent_t ready;
    MRSP_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    MRSP_CUDA(cudaEventRecord(ready, streams[0]));
    const int threads = std::min(256, ((std::max(std::max(V, h), d) + 31) / 32) * 32);
    const size_t smem = sizeof(double) * (2 * d + h);
    for (int w = 0; w < sp_degree; ++w) {
      if (plist[w].empty()) continue;
      MRSP_CUDA(cudaStreamWaitEvent(streams[w], ready, 0));
      toy_prefill_kernel<<<static_cast<unsigned>(plist[w].size()), threads, smem, streams[w]>>>(
          dtheta.p, dctx.p, dpos.p + pos_off[w], dout.p, V, d, h);
      count_launch();
      MRSP_CUDA(cudaGetLastError());
    }
    for (int w = 0; w < sp_degree; ++w) MRSP_CUDA(cudaStreamSynchronize(streams[w]));
    MRSP_CUDA(cudaMemcpy(out, dout.p, sizeof(double) * total * V, cudaMemcpyDeviceToHost));
    cudaEventDestroy(ready);
  });
}
