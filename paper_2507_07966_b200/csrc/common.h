// common.h — status plumbing shared by every translation unit of libmrsp_b200.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include <cstdio>
#include <stdexcept>
#include <string>

#include "mrsp_c.h"

namespace mrsp {

// Exception carrying an mrsp_status; converted at the C-ABI edge.
struct Error : std::runtime_error {
  mrsp_status code;
  Error(mrsp_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& msg);

[[noreturn]] inline void fail(mrsp_status c, const std::string& m) { throw Error(c, m); }

inline void check_cuda(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    (void)cudaGetLastError();  // a failed API call must not resurface at a later launch check
    char buf[512];
    std::snprintf(buf, sizeof(buf), "CUDA error in %s (%s:%d): %s", what, file, line,
                  cudaGetErrorString(e));
    fail(e == cudaErrorMemoryAllocation ? MRSP_OUT_OF_MEMORY : MRSP_CUDA_ERROR, buf);
  }
}

// Runs f, mapping exceptions onto a status + thread-local message.
template <typename F>
mrsp_status guard(F&& f) {
  try {
    f();
    set_last_error("");
    return MRSP_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return MRSP_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return MRSP_RUNTIME_ERROR;
  }
}

// Ensures a CUDA device exists; the product has no CPU fallback.
void require_device();

// Count of kernels this library has launched (evidence for bench.py's gpu_launches).
void count_launch(uint64_t n = 1);

// Programmatic dependent launch for the calling thread's launches (pdl.cuh).
bool pdl_enabled();
void set_pdl(bool on);

// SMs of the current device (grid sizing); 148 on B200.
inline int num_sms() {
  static int n = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  return n;
}

// Query-row split of one kv head's attention over the m SP ranks sharing it
// (HeadSplit::rparts). The work unit is the attention kernel's query block of
// ATTN_ROW_BLOCK rows (two 128-row tiles, one CTA per head). Blocks are dealt
// heaviest first — block b of n sees ~b KV tiles under the causal mask, so
// i = n - 1 - b orders them by descending cost — in a snake 0..m-1, m-1..0, ...
// so the m shares differ by at most one block's cost.
constexpr int ATTN_ROW_BLOCK = 256;

__host__ __device__ inline int attn_row_part(int b, int n_blocks, int m) {
  const int i = n_blocks - 1 - b, r = i / m, p = i - r * m;
  return (r & 1) ? m - 1 - p : p;
}

// Block of the li-th share of part p (< 0: p owns fewer than li + 1 blocks).
__host__ __device__ inline int attn_row_block(int li, int part, int n_blocks, int m) {
  return n_blocks - 1 - (li * m + ((li & 1) ? m - 1 - part : part));
}

}  // namespace mrsp

#define MRSP_CUDA(x) ::mrsp::check_cuda((x), #x, __FILE__, __LINE__)
#define MRSP_REQUIRE(cond, code, msg) \
  do {                                \
    if (!(cond)) ::mrsp::fail(code, msg); \
  } while (0)
