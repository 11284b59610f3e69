// abi_core.cpp — error plumbing, device probe and shard planning.
#include <atomic>
#include <cstring>
#include <string>

#include "common.h"

namespace mrsp {

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

static thread_local bool g_pdl = false;
bool pdl_enabled() { return g_pdl; }
void set_pdl(bool on) { g_pdl = on; }

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

uint64_t mrsp_launch_count(void) { return mrsp::g_launches.load(); }

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

// ---------------------------------------------------------------------------
// Synthetic inputs (mmseq.cpp:58-72, common.hpp:19-79): frames U[-1,1) from
// mt19937_64 seeded by Rng::substream(seed, "video"); delivered as fp32.
#include <random>

namespace {
uint64_t substream_seed(uint64_t base, const char* tag) {
  uint64_t h = 1469598103934665603ull;
  for (const unsigned char* c = reinterpret_cast<const unsigned char*>(tag); *c; ++c) {
    h ^= *c;
    h *= 1099511628211ull;
  }
  uint64_t z = base ^ h;
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
}  // namespace

extern "C" mrsp_status mrsp_gen_video(uint64_t seed, int frames, int feature_dim, float* out) {
  return mrsp::guard([&] {
    MRSP_REQUIRE(frames >= 1, MRSP_INVALID_ARGUMENT, "gen_video: num_frames must be >= 1");
    MRSP_REQUIRE(feature_dim >= 4, MRSP_INVALID_ARGUMENT, "gen_video: feature_dim must be >= 4");
    std::mt19937_64 g(substream_seed(seed, "video"));
    const size_t n = static_cast<size_t>(frames) * static_cast<size_t>(feature_dim);
    for (size_t i = 0; i < n; ++i) {
      const double u = static_cast<double>(g() >> 11) * 0x1.0p-53;
      out[i] = static_cast<float>(2.0 * u - 1.0);
    }
  });
}
