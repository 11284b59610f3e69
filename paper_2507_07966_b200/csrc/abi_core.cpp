// abi_core.cpp — error plumbing, device probe and shard planning.
#include <cstring>
#include <string>

#include "common.h"

namespace mrsp {

static thread_local std::string g_last_error;

void set_last_error(const std::string& msg) { g_last_error = msg; }

void require_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    fail(MRSP_NO_DEVICE,
         "libmrsp_b200: no CUDA device visible; this engine has no CPU fallback");
  }
}

}  // namespace mrsp

extern "C" {

const char* mrsp_last_error(void) { return mrsp::g_last_error.c_str(); }

const char* mrsp_version(void) { return "mrsp_b200 0.1 (sm_100a)"; }

int mrsp_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

// engine.cpp:15-29: base = n / k, the first n % k ranges get one extra item.
mrsp_status mrsp_plan_shards(uint64_t n_items, int sp_degree, uint64_t* ranges) {
  return mrsp::guard([&] {
    MRSP_REQUIRE(sp_degree >= 1, MRSP_INVALID_ARGUMENT, "plan_shards: sp_degree must be >= 1");
    MRSP_REQUIRE(ranges != nullptr, MRSP_INVALID_ARGUMENT, "plan_shards: null output");
    const uint64_t k = static_cast<uint64_t>(sp_degree);
    const uint64_t base = n_items / k, extra = n_items % k;
    uint64_t pos = 0;
    for (uint64_t w = 0; w < k; ++w) {
      const uint64_t len = base + (w < extra ? 1 : 0);
      ranges[2 * w] = pos;
      ranges[2 * w + 1] = pos + len;
      pos += len;
    }
  });
}

}  // extern "C"
