// engine.cu — B200 MR-SP engine: Stage 1 (sharded vision encode -> all-gather
// -> device-resident exactly-once cache) and Stage 2 (packed, sequence-sharded
// Ulysses prefill of policy and reference -> fused LM-head log-probs).
//
// Reference anchors (paths under /root/reference/proj):
//   plan_shards            engine.cpp:15-29   (frame plan and token plan)
//   parallel_encode        engine.cpp:78-101  -> encode_rank() per SP rank
//   all_gather             engine.cpp:132-153 -> NCCL all-gather / in-process
//   EmbeddingCache         engine.cpp:155-197 -> get_or_encode() (same protocol)
//   pad_batch + prefill    engine.cpp:31-43, :103-130, grpo.cpp:44-55
//                          -> packed [video | question | G x Lmax] sequence
//   log_softmax + lp[y]    common.hpp:95-104, grpo.cpp:82-85 -> fused LM head
//   run_step               engine.cpp:203-225 -> mrsp_engine_step
#include "engine.h"

#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <numeric>

#include "attention.h"
#include "common.h"
#include "gemm.h"
#include "misc.h"
#include "pdl.cuh"

namespace mrsp {

// ---------------------------------------------------------------------------
void DevBuf::release() {
  if (p) cudaFree(p);
  p = nullptr;
  bytes = 0;
}
void* DevBuf::ensure(size_t b) {
  if (b <= bytes && p) return p;
  release();
  const size_t nb = std::max<size_t>((b + 255) & ~size_t(255), 256);
  MRSP_CUDA(cudaMalloc(&p, nb));
  bytes = nb;
  return p;
}

namespace {

uint64_t fnv1a(const std::string& s) {
  uint64_t h = 1469598103934665603ull;
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}
uint64_t splitmix(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
uint64_t tensor_key(uint64_t seed, const std::string& name) { return splitmix(seed ^ fnv1a(name)); }

std::vector<std::pair<long, long>> plan(long n, int k) {
  std::vector<std::pair<long, long>> r(k);
  const long base = n / k, extra = n % k;
  long pos = 0;
  for (int w = 0; w < k; ++w) {
    const long len = base + (w < extra ? 1 : 0);
    r[w] = {pos, pos + len};
    pos += len;
  }
  return r;
}

struct Carver {
  uint8_t* base;
  size_t off = 0;
  template <typename T>
  T* take(size_t n) {
    T* p = reinterpret_cast<T*>(base + off);
    off += (n * sizeof(T) + 255) & ~size_t(255);
    return p;
  }
};

}  // namespace

// Ulysses head split for SP rank r of k: contiguous head blocks
// when k <= n_kv; otherwise m = k / n_kv ranks share one kv head (replicated)
// and either split its query-head group with plan_shards (28/4 at SP=8 -> 4+3
// heads: 12.5% attention imbalance; the NCCL transport) or, with row_split,
// each take all of its query heads over 1/m of the query-row blocks, dealt by
// a causal-cost snake (attn_row_part) so the shares are equal to one block.
HeadSplit head_split(int nq, int nkv, int k, int r, bool row_split) {
  HeadSplit h{};
  if (k <= nkv) {
    MRSP_REQUIRE(nkv % k == 0 && nq % k == 0, MRSP_INVALID_ARGUMENT,
                 "ulysses: heads must divide evenly across SP ranks");
    h.q_lo = r * nq / k;
    h.q_hi = (r + 1) * nq / k;
    h.kv_lo = r * nkv / k;
    h.kv_hi = (r + 1) * nkv / k;
    h.q_per_kv = nq / nkv;
  } else {
    MRSP_REQUIRE(k % nkv == 0, MRSP_INVALID_ARGUMENT,
                 "ulysses: SP degree must be a multiple of the kv head count");
    const int m = k / nkv, g = r / m, j = r % m, qpk = nq / nkv;
    if (row_split) {
      h.q_lo = g * qpk;
      h.q_hi = (g + 1) * qpk;
      h.kv_lo = g;
      h.kv_hi = g + 1;
      h.q_per_kv = qpk;
      h.rparts = m;
      h.rpart = j;
      return h;
    }
    const auto p = plan(qpk, m)[j];
    h.q_lo = g * qpk + static_cast<int>(p.first);
    h.q_hi = g * qpk + static_cast<int>(p.second);
    h.kv_lo = g;
    h.kv_hi = g + 1;
    h.q_per_kv = std::max(1, h.q_hi - h.q_lo);
  }
  return h;
}

int vision_head_stride(const mrsp_model_config& c) {
  const char* pad = std::getenv("MRSP_VISION_PAD");
  if (pad && std::atoi(pad) != 0) return 128;
  return c.v_head_dim % 8 == 0 ? c.v_head_dim : 128;
}

// Column blocks of a sequence-shard QKV row [Q heads | K heads | V heads] that
// the destination rank of `hs` owns, as (src col, dst col, width) for Q, K, V;
// the destination stores them as [its Q | its K | its V].
std::array<std::array<int, 3>, 3> ulysses_blocks(int nq, int nkv, const HeadSplit& hs) {
  const int Cq = hs.nq() * 128, Ckv = hs.nkv() * 128;
  return {std::array<int, 3>{hs.q_lo * 128, 0, Cq},
          std::array<int, 3>{nq * 128 + hs.kv_lo * 128, Cq, Ckv},
          std::array<int, 3>{(nq + nkv) * 128 + hs.kv_lo * 128, Cq + Ckv, Ckv}};
}

// ---------------------------------------------------------------------------
Engine::Engine(const mrsp_model_config& cfg, int sp_degree, int proc_rank, int n_procs,
               uint64_t vision_seed, uint64_t policy_seed, uint64_t ref_seed, int with_ref,
               const void* nccl_id)
    : cfg_(cfg), k_(sp_degree), proc_rank_(proc_rank), n_procs_(n_procs) {
  MRSP_REQUIRE(sp_degree >= 1, MRSP_INVALID_ARGUMENT, "WorkerGroup: sp_degree must be >= 1");
  MRSP_REQUIRE(n_procs >= 1 && (n_procs == 1 || n_procs == sp_degree), MRSP_INVALID_ARGUMENT,
               "engine: n_procs must be 1 (virtual ranks) or equal to sp_degree");
  MRSP_REQUIRE(cfg.head_dim == 128, MRSP_INVALID_ARGUMENT, "engine: head_dim must be 128");
  MRSP_REQUIRE(cfg.v_head_dim <= 128 && cfg.v_head_dim * cfg.v_heads == cfg.v_dim,
               MRSP_INVALID_ARGUMENT, "engine: bad vision head geometry");
  MRSP_REQUIRE(cfg.mlp % 128 == 0, MRSP_INVALID_ARGUMENT, "engine: mlp must be a multiple of 128");
  MRSP_REQUIRE(cfg.dim % 8 == 0 && cfg.v_dim % 8 == 0 && cfg.v_mlp % 8 == 0, MRSP_INVALID_ARGUMENT,
               "engine: model dims must be multiples of 8");
  MRSP_REQUIRE(cfg.image_size % cfg.patch == 0, MRSP_INVALID_ARGUMENT,
               "engine: image size must be a multiple of the patch");
  require_device();
  MRSP_CUDA(cudaGetDevice(&device_));
  MRSP_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  if (n_procs > 1) {
    if (nccl_id)
      nccl_ = std::make_unique<Nccl>(n_procs, proc_rank, nccl_id, device_);
    else  // peer memory: mrsp_engine_p2p_export / _import before the first call
      mesh_ = std::make_unique<PeerMesh>(n_procs, proc_rank);
  }
  {
    const char* split = std::getenv("MRSP_ULYSSES_SPLIT");
    row_split_ = !nccl_ && k_ > cfg.n_kv_heads && !(split && std::string(split) == "heads");
  }
  const int local = n_procs > 1 ? 1 : k_;
  ranks_.resize(local);
  for (int i = 0; i < local; ++i) {
    ranks_[i].g = n_procs > 1 ? proc_rank : i;
    ranks_[i].hs = split_of(ranks_[i].g);
  }
  vstride_ = vision_head_stride(cfg);
  float inv[64];
  rope_inv_freq(cfg.rope_theta, inv);  // HF float32 convention (kernels_misc.cu)
  set_rope_inv_freq(inv, stream_);
  build_routes(inv);
  init_weights(vision_seed, policy_seed, ref_seed, with_ref);
  MRSP_CUDA(cudaStreamSynchronize(stream_));
}

// Route of every 128-column head block of a sequence-shard QKV row to the SP
// rank(s) owning that head (a kv head has two owners when SP > n_kv), as
// (rank, destination column) — the static part of the fused all-to-all.
void Engine::build_routes(const float* inv_freq) {
  const int nq = cfg_.n_q_heads, nkv = cfg_.n_kv_heads, nblk = nq + 2 * nkv;
  MRSP_REQUIRE(k_ <= 8, MRSP_INVALID_ARGUMENT, "engine: SP degree <= 8");
  std::vector<int2> route(2 * nblk, make_int2(-1, 0));
  std::vector<int> ld(8, 0);
  auto add = [&](int hb, int rank, int col) {
    int2* r = &route[2 * hb];
    MRSP_REQUIRE(r[1].x < 0, MRSP_INVALID_ARGUMENT, "ulysses: a head block with > 2 owners");
    if (r[0].x < 0) r[0] = make_int2(rank, col);
    else r[1] = make_int2(rank, col);
  };
  if (k_ == 1) {
    for (int hb = 0; hb < nblk; ++hb) add(hb, 0, hb * 128);
    ld[0] = nblk * 128;
  } else if (row_split_) {
    // every rank of kv group g holds [its group's qpk Q heads | K_g | V_g];
    // a Q head block goes to ONE of the group's m ranks, chosen per row block
    // in the QKV epilogue (route (-2, m)); K and V go to all m (route (-3, m))
    const int m = k_ / nkv, qpk = nq / nkv;
    for (int p = 0; p < k_; ++p) ld[p] = (qpk + 2) * 128;
    for (int g = 0; g < nkv; ++g) {
      for (int j = 0; j < qpk; ++j) {
        route[2 * (g * qpk + j)] = make_int2(g * m, j * 128);
        route[2 * (g * qpk + j) + 1] = make_int2(-2, m);
      }
      route[2 * (nq + g)] = make_int2(g * m, qpk * 128);
      route[2 * (nq + g) + 1] = make_int2(-3, m);
      route[2 * (nq + nkv + g)] = make_int2(g * m, (qpk + 1) * 128);
      route[2 * (nq + nkv + g) + 1] = make_int2(-3, m);
    }
  } else {
    for (int p = 0; p < k_; ++p) {
      const HeadSplit hs = split_of(p);
      ld[p] = (hs.nq() + 2 * hs.nkv()) * 128;
      if (hs.nq() == 0) continue;  // no query head: never reads K/V (SP > n_q / q_per_kv)
      for (const auto& blk : ulysses_blocks(nq, nkv, hs))
        for (int c = 0; c < blk[2]; c += 128) add((blk[0] + c) / 128, p, blk[1] + c);
    }
  }
  const size_t off_route = 256, off_ld = off_route + route.size() * sizeof(int2);
  const size_t off_base = (off_ld + 8 * sizeof(int) + 15) & ~size_t(15);
  uint8_t* base = static_cast<uint8_t*>(route_buf_.ensure(off_base + 8 * sizeof(void*)));
  d_inv_freq_ = reinterpret_cast<float*>(base);
  d_route_ = reinterpret_cast<int2*>(base + off_route);
  d_peer_ld_ = reinterpret_cast<int*>(base + off_ld);
  d_peer_base_ = reinterpret_cast<void**>(base + off_base);
  MRSP_CUDA(cudaMemcpy(d_inv_freq_, inv_freq, 64 * sizeof(float), cudaMemcpyHostToDevice));
  MRSP_CUDA(cudaMemcpy(d_route_, route.data(), route.size() * sizeof(int2), cudaMemcpyHostToDevice));
  route_h_ = route;
  MRSP_CUDA(cudaMemcpy(d_peer_ld_, ld.data(), 8 * sizeof(int), cudaMemcpyHostToDevice));
}

Engine::~Engine() {
  if (stream_) cudaStreamSynchronize(stream_);
  for (auto& e : ev_pending_) {
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  for (auto e : ev_pool_) cudaEventDestroy(e);
  ranks_.clear();
  cache_.clear();
  nccl_.reset();
  if (stream_) cudaStreamDestroy(stream_);
}

// Synthetic weights: w = bf16(a * (2u - 1)), u from splitmix64(key + i) (24-bit),
// key = splitmix64(seed ^ fnv1a(name)); restated in oracle/transformer.py.
void Engine::init_weights(uint64_t vseed, uint64_t pseed, uint64_t rseed, int with_ref) {
  const auto& c = cfg_;
  const int T = tokens_per_frame(), kreal = 3 * c.patch * c.patch, kpad = (kreal + 7) / 8 * 8;
  const int vd = c.v_dim, vh = c.v_heads, vhd = c.v_head_dim, vs = vstride_;
  const int vq = vh * vs;
  const int d = c.dim, qkv_rows = (c.n_q_heads + 2 * c.n_kv_heads) * 128;
  has_ref_ = with_ref != 0;
  // size the single weight allocation
  size_t total = 0;
  auto add = [&](size_t n, size_t es) { total += (n * es + 255) & ~size_t(255); };
  add(static_cast<size_t>(vd) * kpad, 2);
  add(vd, 4);
  add(static_cast<size_t>(T) * vd, 4);
  for (int l = 0; l < c.v_layers; ++l) {
    add(vd, 4); add(vd, 4); add(static_cast<size_t>(3) * vq * vd, 2); add(3 * vq, 4);
    add(static_cast<size_t>(vd) * vq, 2); add(vd, 4); add(vd, 4); add(vd, 4);
    add(static_cast<size_t>(c.v_mlp) * vd, 2); add(c.v_mlp, 4);
    add(static_cast<size_t>(vd) * c.v_mlp, 2); add(vd, 4);
  }
  add(vd, 4); add(vd, 4);
  add(static_cast<size_t>(d) * vd, 2); add(d, 4); add(static_cast<size_t>(d) * d, 2); add(d, 4);
  const int n_llm = has_ref_ ? 2 : 1;
  for (int m = 0; m < n_llm; ++m) {
    add(static_cast<size_t>(c.vocab) * d, 2);
    for (int l = 0; l < c.layers; ++l) {
      add(d, 4); add(static_cast<size_t>(qkv_rows) * d, 2); add(qkv_rows, 4);
      add(static_cast<size_t>(d) * c.n_q_heads * 128, 2); add(d, 4);
      add(static_cast<size_t>(2) * c.mlp * d, 2); add(static_cast<size_t>(d) * c.mlp, 2);
    }
    add(d, 4);
    add(static_cast<size_t>(c.vocab) * d, 2);
  }
  wbuf_.ensure(total);
  MRSP_CUDA(cudaMemsetAsync(wbuf_.p, 0, total, stream_));
  Carver cv{static_cast<uint8_t*>(wbuf_.p)};
  cudaStream_t s = stream_;
  auto wscale = [](int fan_in) { return static_cast<float>(std::sqrt(3.0 / fan_in)); };
  const float kBias = 0.03f, kNorm = 0.1f, kPos = 0.1f, kEmbed = static_cast<float>(std::sqrt(3.0));
  auto bf = [&](bf16* dst, size_t n, uint64_t seed, const std::string& name, float a) {
    init_uniform_bf16(dst, n, tensor_key(seed, name), a, s);
  };
  auto f32 = [&](float* dst, size_t n, uint64_t seed, const std::string& name, float a, float off) {
    init_uniform_f32(dst, n, tensor_key(seed, name), a, off, s);
  };
  DevBuf tmp;
  // ---- vision tower
  vis_.patch_w = cv.take<bf16>(static_cast<size_t>(vd) * kpad);
  {
    bf16* t = static_cast<bf16*>(tmp.ensure(static_cast<size_t>(vd) * kreal * 2));
    bf(t, static_cast<size_t>(vd) * kreal, vseed, "vision.patch_w", wscale(kreal));
    MRSP_CUDA(cudaMemcpy2DAsync(vis_.patch_w, kpad * 2, t, kreal * 2, kreal * 2, vd,
                                cudaMemcpyDeviceToDevice, s));
  }
  vis_.patch_b = cv.take<float>(vd);
  f32(vis_.patch_b, vd, vseed, "vision.patch_b", kBias, 0.f);
  vis_.pos = cv.take<float>(static_cast<size_t>(T) * vd);
  f32(vis_.pos, static_cast<size_t>(T) * vd, vseed, "vision.pos", kPos, 0.f);
  vis_.layers.resize(c.v_layers);
  for (int l = 0; l < c.v_layers; ++l) {
    auto& L = vis_.layers[l];
    const std::string p = "vision." + std::to_string(l) + ".";
    L.ln1_w = cv.take<float>(vd); f32(L.ln1_w, vd, vseed, p + "ln1_w", kNorm, 1.f);
    L.ln1_b = cv.take<float>(vd); f32(L.ln1_b, vd, vseed, p + "ln1_b", kBias, 0.f);
    // QKV / O with head stride vs (vs > vhd: zero rows / columns)
    L.wqkv = cv.take<bf16>(static_cast<size_t>(3) * vq * vd);
    {
      bf16* t = static_cast<bf16*>(tmp.ensure(static_cast<size_t>(3) * vd * vd * 2));
      bf(t, static_cast<size_t>(3) * vd * vd, vseed, p + "wqkv", wscale(vd));
      for (int part = 0; part < 3; ++part)
        for (int h = 0; h < vh; ++h)
          MRSP_CUDA(cudaMemcpyAsync(L.wqkv + (static_cast<size_t>(part) * vq + h * vs) * vd,
                                    t + (static_cast<size_t>(part) * vd + h * vhd) * vd,
                                    static_cast<size_t>(vhd) * vd * 2, cudaMemcpyDeviceToDevice, s));
    }
    L.bqkv = cv.take<float>(3 * vq);
    {
      float* t = static_cast<float*>(tmp.ensure(static_cast<size_t>(3) * vd * 4));
      f32(t, 3 * vd, vseed, p + "bqkv", kBias, 0.f);
      for (int part = 0; part < 3; ++part)
        for (int h = 0; h < vh; ++h)
          MRSP_CUDA(cudaMemcpyAsync(L.bqkv + part * vq + h * vs, t + part * vd + h * vhd, vhd * 4,
                                    cudaMemcpyDeviceToDevice, s));
    }
    L.wo = cv.take<bf16>(static_cast<size_t>(vd) * vq);
    {
      bf16* t = static_cast<bf16*>(tmp.ensure(static_cast<size_t>(vd) * vd * 2));
      bf(t, static_cast<size_t>(vd) * vd, vseed, p + "wo", wscale(vd));
      for (int h = 0; h < vh; ++h)
        MRSP_CUDA(cudaMemcpy2DAsync(L.wo + h * vs, static_cast<size_t>(vq) * 2, t + h * vhd,
                                    static_cast<size_t>(vd) * 2, vhd * 2, vd,
                                    cudaMemcpyDeviceToDevice, s));
    }
    L.bo = cv.take<float>(vd); f32(L.bo, vd, vseed, p + "bo", kBias, 0.f);
    L.ln2_w = cv.take<float>(vd); f32(L.ln2_w, vd, vseed, p + "ln2_w", kNorm, 1.f);
    L.ln2_b = cv.take<float>(vd); f32(L.ln2_b, vd, vseed, p + "ln2_b", kBias, 0.f);
    L.w1 = cv.take<bf16>(static_cast<size_t>(c.v_mlp) * vd);
    bf(L.w1, static_cast<size_t>(c.v_mlp) * vd, vseed, p + "w1", wscale(vd));
    L.b1 = cv.take<float>(c.v_mlp); f32(L.b1, c.v_mlp, vseed, p + "b1", kBias, 0.f);
    L.w2 = cv.take<bf16>(static_cast<size_t>(vd) * c.v_mlp);
    bf(L.w2, static_cast<size_t>(vd) * c.v_mlp, vseed, p + "w2", wscale(c.v_mlp));
    L.b2 = cv.take<float>(vd); f32(L.b2, vd, vseed, p + "b2", kBias, 0.f);
  }
  vis_.post_w = cv.take<float>(vd); f32(vis_.post_w, vd, vseed, "vision.post_w", kNorm, 1.f);
  vis_.post_b = cv.take<float>(vd); f32(vis_.post_b, vd, vseed, "vision.post_b", kBias, 0.f);
  vis_.p1_w = cv.take<bf16>(static_cast<size_t>(d) * vd);
  bf(vis_.p1_w, static_cast<size_t>(d) * vd, vseed, "proj.w1", wscale(vd));
  vis_.p1_b = cv.take<float>(d); f32(vis_.p1_b, d, vseed, "proj.b1", kBias, 0.f);
  vis_.p2_w = cv.take<bf16>(static_cast<size_t>(d) * d);
  bf(vis_.p2_w, static_cast<size_t>(d) * d, vseed, "proj.w2", wscale(d));
  vis_.p2_b = cv.take<float>(d); f32(vis_.p2_b, d, vseed, "proj.b2", kBias, 0.f);
  // ---- LLMs
  for (int m = 0; m < n_llm; ++m) {
    auto& W = llm_[m];
    const uint64_t seed = m == 0 ? pseed : rseed;
    const std::string pre = m == 0 ? "policy." : "ref.";
    W.embed = cv.take<bf16>(static_cast<size_t>(c.vocab) * d);
    bf(W.embed, static_cast<size_t>(c.vocab) * d, seed, pre + "embed", kEmbed);
    W.layers.resize(c.layers);
    for (int l = 0; l < c.layers; ++l) {
      auto& L = W.layers[l];
      const std::string p = pre + std::to_string(l) + ".";
      L.attn_norm = cv.take<float>(d); f32(L.attn_norm, d, seed, p + "attn_norm", kNorm, 1.f);
      L.wqkv = cv.take<bf16>(static_cast<size_t>(qkv_rows) * d);
      bf(L.wqkv, static_cast<size_t>(qkv_rows) * d, seed, p + "wqkv", wscale(d));
      L.bqkv = cv.take<float>(qkv_rows); f32(L.bqkv, qkv_rows, seed, p + "bqkv", kBias, 0.f);
      L.wo = cv.take<bf16>(static_cast<size_t>(d) * c.n_q_heads * 128);
      bf(L.wo, static_cast<size_t>(d) * c.n_q_heads * 128, seed, p + "wo", wscale(c.n_q_heads * 128));
      L.mlp_norm = cv.take<float>(d); f32(L.mlp_norm, d, seed, p + "mlp_norm", kNorm, 1.f);
      L.wgu = cv.take<bf16>(static_cast<size_t>(2) * c.mlp * d);
      {
        // interleave [gate | up] in 128-row blocks for the SwiGLU epilogue
        const size_t n1 = static_cast<size_t>(c.mlp) * d;
        bf16* t = static_cast<bf16*>(tmp.ensure(n1 * 2));
        bf(t, n1, seed, p + "w_gate", wscale(d));
        MRSP_CUDA(cudaMemcpy2DAsync(L.wgu, static_cast<size_t>(256) * d * 2, t,
                                    static_cast<size_t>(128) * d * 2, static_cast<size_t>(128) * d * 2,
                                    c.mlp / 128, cudaMemcpyDeviceToDevice, s));
        MRSP_CUDA(cudaStreamSynchronize(s));
        bf(t, n1, seed, p + "w_up", wscale(d));
        MRSP_CUDA(cudaMemcpy2DAsync(L.wgu + static_cast<size_t>(128) * d,
                                    static_cast<size_t>(256) * d * 2, t,
                                    static_cast<size_t>(128) * d * 2, static_cast<size_t>(128) * d * 2,
                                    c.mlp / 128, cudaMemcpyDeviceToDevice, s));
        MRSP_CUDA(cudaStreamSynchronize(s));
      }
      L.wdown = cv.take<bf16>(static_cast<size_t>(d) * c.mlp);
      bf(L.wdown, static_cast<size_t>(d) * c.mlp, seed, p + "w_down", wscale(c.mlp));
    }
    W.final_norm = cv.take<float>(d); f32(W.final_norm, d, seed, pre + "final_norm", kNorm, 1.f);
    W.lm_head = cv.take<bf16>(static_cast<size_t>(c.vocab) * d);
    bf(W.lm_head, static_cast<size_t>(c.vocab) * d, seed, pre + "lm_head", wscale(d));
  }
  if (!has_ref_) llm_[1] = llm_[0];
  MRSP_CUDA(cudaStreamSynchronize(s));
}

// ---------------------------------------------------------------------------
void Engine::prof_begin(int cls, cudaEvent_t* a) {
  (void)cls;
  if (!prof_) return;
  if (ev_pool_.empty()) {
    cudaEvent_t e;
    MRSP_CUDA(cudaEventCreate(&e));
    ev_pool_.push_back(e);
  }
  *a = ev_pool_.back();
  ev_pool_.pop_back();
  MRSP_CUDA(cudaEventRecord(*a, stream_));
}
void Engine::prof_end(int cls, cudaEvent_t a) {
  if (!prof_) return;
  cudaEvent_t b;
  if (ev_pool_.empty()) {
    MRSP_CUDA(cudaEventCreate(&b));
  } else {
    b = ev_pool_.back();
    ev_pool_.pop_back();
  }
  MRSP_CUDA(cudaEventRecord(b, stream_));
  ev_pending_.push_back({cls, a, b});
}
void Engine::prof_collect() {
  if (ev_pending_.empty()) return;
  MRSP_CUDA(cudaStreamSynchronize(stream_));
  for (auto& e : ev_pending_) {
    float ms = 0;
    MRSP_CUDA(cudaEventElapsedTime(&ms, e.a, e.b));
    prof_ms_[e.cls] += ms;
    prof_n_[e.cls] += 1;
    ev_pool_.push_back(e.a);
    ev_pool_.push_back(e.b);
  }
  ev_pending_.clear();
}
void Engine::set_profiling(bool on) {
  prof_collect();
  prof_ = on;
  if (on) {
    for (int i = 0; i < kProfClasses; ++i) {
      prof_ms_[i] = 0;
      prof_n_[i] = 0;
    }
  }
}
void Engine::profile_read(int cls, double* ms, long* launches) {
  prof_collect();
  *ms = prof_ms_[cls];
  *launches = prof_n_[cls];
}

// RAII timing scope for one kernel class.

// ---------------------------------------------------------------------------
// Stage 1 for one SP rank: frames [fb, fe) -> projector output rows.
void Engine::encode_rank(RankCtx& R, const float* pixels, bool on_device, int F, long fb, long fe,
                         bf16* out) {
  (void)F;
  const auto& c = cfg_;
  const int nf = static_cast<int>(fe - fb);
  if (nf <= 0) return;
  const int T = tokens_per_frame(), S = c.image_size, P = c.patch;
  const int kreal = 3 * P * P, kpad = (kreal + 7) / 8 * 8;
  const int vd = c.v_dim, vs = vstride_, vq = c.v_heads * vs, ntok = nf * T;
  cudaStream_t s = stream_;
  const size_t frame_px = static_cast<size_t>(3) * S * S;
  Prof pv(*this, P_VISION);
  float* pix = static_cast<float*>(R.pix.ensure(static_cast<size_t>(nf) * frame_px * 4));
  MRSP_CUDA(cudaMemcpyAsync(pix, pixels + static_cast<size_t>(fb) * frame_px,
                            static_cast<size_t>(nf) * frame_px * 4,
                            on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
  bf16* patches = static_cast<bf16*>(R.patches.ensure(static_cast<size_t>(ntok) * kpad * 2));
  patchify(pix, patches, nf, S, S, P, kpad, s);
  float* vh = static_cast<float*>(R.vh.ensure(static_cast<size_t>(ntok) * vd * 4));
  bf16* xn = static_cast<bf16*>(R.vxn.ensure(static_cast<size_t>(ntok) * vd * 2));
  bf16* qkv = static_cast<bf16*>(R.vqkv.ensure(static_cast<size_t>(ntok) * 3 * vq * 2));
  bf16* o = static_cast<bf16*>(R.vo.ensure(static_cast<size_t>(ntok) * vq * 2));
  bf16* mid = static_cast<bf16*>(
      R.vmid.ensure(static_cast<size_t>(ntok) * std::max(c.v_mlp, c.dim) * 2));
  broadcast_rows(vis_.pos, vh, ntok, T, vd, s);
  gemm_bf16({patches, vis_.patch_w, nullptr, ntok, vd, kpad, kpad, kpad, 0, GEMM_EPI_RESID_F32,
             vis_.patch_b, vh, vd},
            s);
  const float vscale = 1.0f / std::sqrt(static_cast<float>(c.v_head_dim));
  for (const auto& L : vis_.layers) {
    layernorm(vh, vd, L.ln1_w, L.ln1_b, xn, vd, ntok, vd, c.ln_eps, s);
    gemm_bf16({xn, L.wqkv, qkv, ntok, 3 * vq, vd, vd, vd, 3 * vq, GEMM_EPI_BIAS_BF16, L.bqkv,
               nullptr, 0},
              s);
    AttnParams ap{qkv, 3 * vq, 0, qkv, 3 * vq, vq, qkv, 3 * vq, 2 * vq, o, vq, 0, ntok,
                  c.v_heads, 1, vscale, ATTN_BLOCK_DIAG, 0, 0, T};
    ap.hstride = vs;
    attention_fwd(ap, s);
    gemm_bf16({o, L.wo, nullptr, ntok, vd, vq, vq, vq, 0, GEMM_EPI_RESID_F32, L.bo, vh, vd}, s);
    layernorm(vh, vd, L.ln2_w, L.ln2_b, xn, vd, ntok, vd, c.ln_eps, s);
    gemm_bf16({xn, L.w1, mid, ntok, c.v_mlp, vd, vd, vd, c.v_mlp, GEMM_EPI_BIAS_GELU_BF16, L.b1,
               nullptr, 0},
              s);
    gemm_bf16({mid, L.w2, nullptr, ntok, vd, c.v_mlp, c.v_mlp, c.v_mlp, 0, GEMM_EPI_RESID_F32,
               L.b2, vh, vd},
              s);
  }
  layernorm(vh, vd, vis_.post_w, vis_.post_b, xn, vd, ntok, vd, c.ln_eps, s);
  gemm_bf16({xn, vis_.p1_w, mid, ntok, c.dim, vd, vd, vd, c.dim, GEMM_EPI_BIAS_GELU_BF16,
             vis_.p1_b, nullptr, 0},
            s);
  gemm_bf16({mid, vis_.p2_w, out, ntok, c.dim, c.dim, c.dim, c.dim, c.dim, GEMM_EPI_BIAS_BF16,
             vis_.p2_b, nullptr, 0},
            s);
  encoder_invocations.fetch_add(static_cast<uint64_t>(nf), std::memory_order_relaxed);
}

// Device buffer for a cache entry's embeddings: an evicted entry's buffer of
// the same size is reused once nothing references it (cudaMalloc / cudaFree of
// a ~1 GB buffer per fresh video stalls the stream); MRSP_CACHE_POOL=0 turns
// the recycling off. Called under run_mu_.
std::shared_ptr<DevBuf> Engine::entry_buffer(size_t bytes) {
  static const bool pool_on = [] {
    const char* v = std::getenv("MRSP_CACHE_POOL");
    return !(v && std::atoi(v) == 0);
  }();
  if (pool_on) {
    for (auto& b : entry_pool_)
      if (b.use_count() == 1 && b->bytes >= bytes && b->bytes <= bytes + (bytes >> 3)) return b;
  }
  auto b = std::make_shared<DevBuf>();
  b->ensure(bytes);
  if (pool_on) {
    if (entry_pool_.size() >= 6) {  // drop a buffer nobody holds, else do not pool
      for (auto it = entry_pool_.begin(); it != entry_pool_.end(); ++it)
        if (it->use_count() == 1) {
          entry_pool_.erase(it);
          break;
        }
    }
    if (entry_pool_.size() < 6) entry_pool_.push_back(b);
  }
  return b;
}

std::shared_ptr<CacheEntry> Engine::get_or_encode(const std::string& id, const float* pixels,
                                                  int F, bool on_device, bool use_cache,
                                                  bool* hit) {
  MRSP_REQUIRE(F >= 1, MRSP_INVALID_ARGUMENT, "gen_video: num_frames must be >= 1");
  std::shared_ptr<CacheEntry> entry;
  bool filler = true;
  if (use_cache) {
    std::lock_guard<std::mutex> lock(cache_mu_);
    auto it = cache_.find(id);
    if (it == cache_.end()) {
      entry = std::make_shared<CacheEntry>();
      entry->seq = ++cache_seq_;
      cache_.emplace(id, entry);
      cache_misses.fetch_add(1, std::memory_order_relaxed);
      if (cache_capacity > 0) {
        while (static_cast<int>(cache_.size()) > cache_capacity) {
          auto oldest = std::min_element(cache_.begin(), cache_.end(), [](auto& a, auto& b) {
            return a.second->seq < b.second->seq;
          });
          cache_.erase(oldest);
        }
      }
    } else {
      entry = it->second;
      filler = false;
      cache_hits.fetch_add(1, std::memory_order_relaxed);
    }
  } else {
    entry = std::make_shared<CacheEntry>();
  }
  *hit = !filler;
  if (!filler) {
    std::unique_lock<std::mutex> lock(entry->m);
    entry->cv.wait(lock, [&] { return entry->ready; });
    if (entry->failed) fail(MRSP_RUNTIME_ERROR, entry->error);
    return entry;
  }
  try {
    std::lock_guard<std::mutex> run(run_mu_);
    const int T = tokens_per_frame(), d = cfg_.dim;
    const auto fplan = plan(F, k_);
    const size_t row_bytes = static_cast<size_t>(T) * d * 2;  // one frame's embeddings
    auto emb = entry_buffer(static_cast<size_t>(F) * row_bytes);
    bf16* full = static_cast<bf16*>(emb->p);
    if (mesh_) {
      // one process per GPU over peer memory: encode this rank's frames, then
      // copy-engine P2P writes of the slice into every rank's landing buffer
      MRSP_REQUIRE(mesh_->ready() && F <= mesh_->caps().frames, MRSP_INVALID_ARGUMENT,
                   "p2p: mesh not set up or video longer than its frame capacity");
      RankCtx& R = ranks_[0];
      const auto [fb, fe] = fplan[R.g];
      uint8_t* sendb = static_cast<uint8_t*>(R.send.ensure(std::max<long>(fe - fb, 1) * row_bytes));
      encode_rank(R, pixels, on_device, F, fb, fe, reinterpret_cast<bf16*>(sendb));
      Prof pc(*this, P_COMM);
      mesh_->barrier(stream_);  // every rank has copied the previous video out
      if (fe > fb)
        for (int p = 0; p < k_; ++p)
          MRSP_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(mesh_->emb(p)) + fb * row_bytes, sendb,
                                    (fe - fb) * row_bytes, cudaMemcpyDeviceToDevice, stream_));
      mesh_->barrier(stream_);
      MRSP_CUDA(cudaMemcpyAsync(full, mesh_->emb(R.g), F * row_bytes, cudaMemcpyDeviceToDevice,
                                stream_));
    } else if (!nccl_) {
      // virtual ranks share this device: each rank's projector writes its
      // slice of the gathered buffer directly (the in-process all-gather)
      for (auto& R : ranks_) {
        const auto [fb, fe] = fplan[R.g];
        encode_rank(R, pixels, on_device, F, fb, fe, full + static_cast<size_t>(fb) * T * d);
      }
    } else {
      RankCtx& R = ranks_[0];
      const auto [fb, fe] = fplan[R.g];
      const long chunk_frames = (F + k_ - 1) / k_;
      const size_t chunk = chunk_frames * row_bytes;
      uint8_t* sendb = static_cast<uint8_t*>(R.send.ensure(chunk));
      uint8_t* recvb = static_cast<uint8_t*>(R.recv.ensure(chunk * k_));
      encode_rank(R, pixels, on_device, F, fb, fe, reinterpret_cast<bf16*>(sendb));
      {
        Prof pc(*this, P_COMM);
        nccl_->all_gather(sendb, recvb, chunk, stream_);
      }
      for (int w = 0; w < k_; ++w) {
        const auto [b, e] = fplan[w];
        if (e > b)
          MRSP_CUDA(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(full) + b * row_bytes,
                                    recvb + w * chunk, (e - b) * row_bytes,
                                    cudaMemcpyDeviceToDevice, stream_));
      }
    }
    // reference accounting: values x (sp - 1) x bytes per value (engine.cpp:149-151)
    gather_bytes.fetch_add(static_cast<uint64_t>(F) * T * d * (k_ - 1) * 2,
                           std::memory_order_relaxed);
    MRSP_CUDA(cudaStreamSynchronize(stream_));
    prof_collect();
    {
      std::lock_guard<std::mutex> lock(entry->m);
      entry->emb = emb;
      entry->n_frames = F;
      entry->ready = true;
    }
    entry->cv.notify_all();
  } catch (const std::exception& ex) {
    {
      std::lock_guard<std::mutex> lock(entry->m);
      entry->failed = true;
      entry->error = ex.what();
      entry->ready = true;
    }
    entry->cv.notify_all();
    if (use_cache) {
      std::lock_guard<std::mutex> lock(cache_mu_);
      auto it = cache_.find(id);
      if (it != cache_.end() && it->second == entry) cache_.erase(it);
    }
    throw;
  }
  return entry;
}

// ---------------------------------------------------------------------------
// Ulysses all-to-all: sequence shards [n_r, Cqkv] -> head shards [L, C_r].
void Engine::a2a_forward(int L) {
  (void)L;
  const auto& c = cfg_;
  const int nq = c.n_q_heads, nkv = c.n_kv_heads, Cqkv = (nq + 2 * nkv) * 128;
  Prof pc(*this, P_COMM);
  auto col_blocks = [&](const HeadSplit& hs) { return ulysses_blocks(nq, nkv, hs); };
  if (!nccl_) {
    for (auto& dst : ranks_) {
      const int Cr = (dst.hs.nq() + 2 * dst.hs.nkv()) * 128;
      bf16* qh = dst.qh.as<bf16>();
      for (auto& src : ranks_) {
        const long n = src.e - src.b;
        if (n <= 0) continue;
        for (auto& blk : col_blocks(dst.hs)) {
          if (blk[2] == 0) continue;
          MRSP_CUDA(cudaMemcpy2DAsync(qh + static_cast<size_t>(src.b) * Cr + blk[1],
                                      static_cast<size_t>(Cr) * 2,
                                      src.qkv.as<bf16>() + blk[0], static_cast<size_t>(Cqkv) * 2,
                                      static_cast<size_t>(blk[2]) * 2, n, cudaMemcpyDeviceToDevice,
                                      stream_));
          if (&src != &dst) a2a_bytes.fetch_add(static_cast<uint64_t>(n) * blk[2] * 2);
        }
      }
    }
    return;
  }
  RankCtx& me = ranks_[0];
  const long n_me = me.e - me.b;
  const int Cme = (me.hs.nq() + 2 * me.hs.nkv()) * 128;
  // pack per-peer send blocks [n_me, C_peer]
  std::vector<size_t> soff(k_ + 1, 0);
  std::vector<HeadSplit> hs(k_);
  for (int p = 0; p < k_; ++p) {
    hs[p] = split_of(p);
    soff[p + 1] = soff[p] + static_cast<size_t>(n_me) * (hs[p].nq() + 2 * hs[p].nkv()) * 128;
  }
  bf16* sendb = static_cast<bf16*>(me.send.ensure(std::max<size_t>(soff[k_], 1) * 2));
  for (int p = 0; p < k_; ++p) {
    const int Cp = (hs[p].nq() + 2 * hs[p].nkv()) * 128;
    for (auto& blk : col_blocks(hs[p])) {
      if (blk[2] == 0 || n_me == 0) continue;
      bf16* dst = p == me.g ? me.qh.as<bf16>() + static_cast<size_t>(me.b) * Cme + blk[1]
                            : sendb + soff[p] + blk[1];
      MRSP_CUDA(cudaMemcpy2DAsync(dst, static_cast<size_t>(Cp) * 2, me.qkv.as<bf16>() + blk[0],
                                  static_cast<size_t>(Cqkv) * 2, static_cast<size_t>(blk[2]) * 2,
                                  n_me, cudaMemcpyDeviceToDevice, stream_));
    }
  }
  nccl_->group_start();
  for (int p = 0; p < k_; ++p) {
    if (p == me.g) continue;
    const size_t sb = (soff[p + 1] - soff[p]) * 2;
    if (sb) nccl_->send(sendb + soff[p], sb, p, stream_);
    const long b = token_b_[p], e = token_e_[p];
    const size_t rb = static_cast<size_t>(e - b) * Cme * 2;
    if (rb) nccl_->recv(me.qh.as<bf16>() + static_cast<size_t>(b) * Cme, rb, p, stream_);
    a2a_bytes.fetch_add(sb);
  }
  nccl_->group_end();
}

// Head shards [L, nq_r*128] -> sequence shards [n_r, nq*128].
void Engine::a2a_backward(int L) {
  (void)L;
  const int nq = cfg_.n_q_heads, Cq = nq * 128;
  Prof pc(*this, P_COMM);
  if (!nccl_) {
    for (auto& src : ranks_) {
      const int Cs = src.hs.nq() * 128;
      if (Cs == 0) continue;
      for (auto& dst : ranks_) {
        const long n = dst.e - dst.b;
        if (n <= 0) continue;
        MRSP_CUDA(cudaMemcpy2DAsync(dst.ol.as<bf16>() + src.hs.q_lo * 128,
                                    static_cast<size_t>(Cq) * 2,
                                    src.oh.as<bf16>() + static_cast<size_t>(dst.b) * Cs,
                                    static_cast<size_t>(Cs) * 2, static_cast<size_t>(Cs) * 2, n,
                                    cudaMemcpyDeviceToDevice, stream_));
        if (&src != &dst) a2a_bytes.fetch_add(static_cast<uint64_t>(n) * Cs * 2);
      }
    }
    return;
  }
  RankCtx& me = ranks_[0];
  const long n_me = me.e - me.b;
  const int Cme = me.hs.nq() * 128;
  std::vector<HeadSplit> hs(k_);
  std::vector<size_t> roff(k_ + 1, 0);
  for (int p = 0; p < k_; ++p) {
    hs[p] = split_of(p);
    roff[p + 1] = roff[p] + static_cast<size_t>(n_me) * hs[p].nq() * 128;
  }
  bf16* recvb = static_cast<bf16*>(me.recv.ensure(std::max<size_t>(roff[k_], 1) * 2));
  nccl_->group_start();
  for (int p = 0; p < k_; ++p) {
    if (p == me.g) continue;
    const long b = token_b_[p], e = token_e_[p];
    const size_t sb = static_cast<size_t>(e - b) * Cme * 2;
    if (sb) nccl_->send(me.oh.as<bf16>() + static_cast<size_t>(b) * Cme, sb, p, stream_);
    const size_t rb = (roff[p + 1] - roff[p]) * 2;
    if (rb) nccl_->recv(recvb + roff[p], rb, p, stream_);
    a2a_bytes.fetch_add(sb);
  }
  nccl_->group_end();
  for (int p = 0; p < k_; ++p) {
    const int Cp = hs[p].nq() * 128;
    if (Cp == 0 || n_me == 0) continue;
    const bf16* src = p == me.g ? me.oh.as<bf16>() + static_cast<size_t>(me.b) * Cme : recvb + roff[p];
    MRSP_CUDA(cudaMemcpy2DAsync(me.ol.as<bf16>() + hs[p].q_lo * 128, static_cast<size_t>(Cq) * 2,
                                src, static_cast<size_t>(Cp) * 2, static_cast<size_t>(Cp) * 2, n_me,
                                cudaMemcpyDeviceToDevice, stream_));
  }
}

// ---------------------------------------------------------------------------
// Host-side pad_batch semantics for one GRPO group: validation, token upload
// (shared by both passes), the token plan and each shard's scored positions.
void Engine::prepare_group(const CacheEntry& emb, const int32_t* question, int n_q,
                           const int32_t* resp, const int32_t* lengths, int G, int Lmax) {
  const auto& c = cfg_;
  MRSP_REQUIRE(G >= 1, MRSP_INVALID_ARGUMENT, "pad_batch: empty batch");
  MRSP_REQUIRE(Lmax >= 1 && n_q >= 0, MRSP_INVALID_ARGUMENT, "prefill: bad lengths");
  const int T = tokens_per_frame(), d = c.dim;
  GroupState& g = grp_;
  g.n_q = n_q;
  g.G = G;
  g.Lmax = Lmax;
  g.n_frame_tok = static_cast<long>(emb.n_frames) * T;
  g.Lp = g.n_frame_tok + n_q;
  g.Ltot = g.Lp + static_cast<long>(G) * Lmax;
  MRSP_REQUIRE(g.Ltot < (1L << 31), MRSP_INVALID_ARGUMENT, "prefill: sequence too long");
  std::vector<long> row_off(G + 1, 0);
  for (int r = 0; r < G; ++r) {
    MRSP_REQUIRE(lengths[r] >= 0 && lengths[r] <= Lmax, MRSP_INVALID_ARGUMENT,
                 "prefill: row longer than Lmax");
    row_off[r + 1] = row_off[r] + lengths[r];
    for (int j = 0; j < lengths[r]; ++j)
      MRSP_REQUIRE(resp[static_cast<size_t>(r) * Lmax + j] >= 0 &&
                       resp[static_cast<size_t>(r) * Lmax + j] < c.vocab,
                   MRSP_INVALID_ARGUMENT, "step_logits: prev token out of range");
  }
  for (int i = 0; i < n_q; ++i)
    MRSP_REQUIRE(question[i] >= 0 && question[i] < c.vocab, MRSP_INVALID_ARGUMENT,
                 "context_vector: token out of range");
  g.total_scored = row_off[G];
  const auto tplan = plan(g.Ltot, k_);
  token_b_.resize(k_);
  token_e_.resize(k_);
  for (int w = 0; w < k_; ++w) {
    token_b_[w] = tplan[w].first;
    token_e_[w] = tplan[w].second;
  }
  cudaStream_t s = stream_;
  const size_t tok_ints = static_cast<size_t>(n_q) + static_cast<size_t>(G) * Lmax + G;
  // [question | resp | lengths] ints, then 4 full-length float vectors
  int32_t* dtok = static_cast<int32_t*>(io_.ensure(tok_ints * 4 + (4 * g.total_scored + 64) * 4));
  MRSP_CUDA(cudaMemcpyAsync(dtok, question, static_cast<size_t>(n_q) * 4, cudaMemcpyHostToDevice, s));
  MRSP_CUDA(cudaMemcpyAsync(dtok + n_q, resp, static_cast<size_t>(G) * Lmax * 4,
                            cudaMemcpyHostToDevice, s));
  MRSP_CUDA(cudaMemcpyAsync(dtok + n_q + static_cast<size_t>(G) * Lmax, lengths,
                            static_cast<size_t>(G) * 4, cudaMemcpyHostToDevice, s));
  g.d_question = dtok;
  g.d_resp = dtok + n_q;
  g.d_len = dtok + n_q + static_cast<size_t>(G) * Lmax;
  g.full = reinterpret_cast<float*>(dtok + tok_ints);  // 4 x (total_scored + 16)
  g.stride = g.total_scored + 16;
  MRSP_CUDA(cudaMemsetAsync(g.full, 0, static_cast<size_t>(4 * g.stride) * 4, s));
  const int Cqkv = (c.n_q_heads + 2 * c.n_kv_heads) * 128, Cq = c.n_q_heads * 128;
  for (auto& R : ranks_) {
    R.b = tplan[R.g].first;
    R.e = tplan[R.g].second;
    const long n = R.e - R.b;
    // scored positions of this shard: row region, j < len (the prev token of
    // position j is read only for j < len, engine.cpp:124 -> pad_reads == 0)
    std::vector<int32_t> idx, tgt, slot;
    for (long p = std::max(R.b, g.Lp); p < R.e; ++p) {
      const long q = p - g.Lp;
      const int r = static_cast<int>(q / Lmax), j = static_cast<int>(q % Lmax);
      if (j < lengths[r]) {
        idx.push_back(static_cast<int32_t>(p - R.b));
        tgt.push_back(resp[static_cast<size_t>(r) * Lmax + j]);
        slot.push_back(static_cast<int32_t>(row_off[r] + j));
      }
    }
    R.n_scored = static_cast<int>(idx.size());
    R.sc_lo = slot.empty() ? 0 : slot[0];  // scored tokens are slot-ordered by position
    {  // this rank's LM-head slice and its [targets | slots]
      if (spread_lm()) {
        const auto sp = plan(g.total_scored, k_)[R.g];
        R.lm_lo = static_cast<long>(sp.first);
        R.lm_n = static_cast<int>(sp.second - sp.first);
      } else {
        R.lm_lo = R.sc_lo;
        R.lm_n = R.n_scored;
      }
      std::vector<int32_t> lm(2 * static_cast<size_t>(R.lm_n));
      for (int i = 0, r = 0; i < R.lm_n; ++i) {
        const long sl = R.lm_lo + i;
        while (row_off[r + 1] <= sl) ++r;
        lm[i] = resp[static_cast<size_t>(r) * Lmax + (sl - row_off[r])];
        lm[R.lm_n + i] = static_cast<int32_t>(sl);
      }
      int32_t* dl = static_cast<int32_t*>(R.lm_idx.ensure((lm.size() + 1) * 4));
      if (!lm.empty()) {
        MRSP_CUDA(cudaMemcpyAsync(dl, lm.data(), lm.size() * 4, cudaMemcpyHostToDevice, s));
        MRSP_CUDA(cudaStreamSynchronize(s));
      }
      if (spread_lm() && !mesh_)
        R.lmx.ensure(static_cast<size_t>(2) * std::max(R.lm_n, 1) * d * 2);
    }
    int32_t* di = static_cast<int32_t*>(R.scored_idx.ensure((idx.size() + 1) * 4 * 3));
    if (!idx.empty()) {
      MRSP_CUDA(cudaMemcpyAsync(di, idx.data(), idx.size() * 4, cudaMemcpyHostToDevice, s));
      MRSP_CUDA(cudaMemcpyAsync(di + idx.size(), tgt.data(), idx.size() * 4, cudaMemcpyHostToDevice, s));
      MRSP_CUDA(cudaMemcpyAsync(di + 2 * idx.size(), slot.data(), idx.size() * 4,
                                cudaMemcpyHostToDevice, s));
      MRSP_CUDA(cudaStreamSynchronize(s));  // host vectors go out of scope
    }
    const size_t nn = static_cast<size_t>(std::max(n, 1L));
    R.h.ensure(nn * d * 4);
    R.xn.ensure(nn * d * 2);
    R.qkv.ensure(nn * Cqkv * 2);
    if (mesh_) {
      MRSP_REQUIRE(mesh_->ready() && g.Ltot <= mesh_->caps().tokens && n <= mesh_->caps().shard &&
                       g.total_scored <= mesh_->caps().scored,
                   MRSP_INVALID_ARGUMENT, "p2p: group exceeds the exported capacities");
    } else {
      R.ol.ensure(nn * Cq * 2);
    }
    R.act.ensure(nn * c.mlp * 2);
    R.pos.ensure(nn * 4);
    R.pad.ensure(nn);
    if (k_ > 1 && !mesh_) {
      R.qh.ensure(static_cast<size_t>(g.Ltot) * (R.hs.nq() + 2 * R.hs.nkv()) * 128 * 2);
      R.oh.ensure(static_cast<size_t>(g.Ltot) * std::max(R.hs.nq(), 1) * 128 * 2);
    }
    R.xs.ensure(static_cast<size_t>(std::max(R.n_scored, 1)) * d * 2);
    R.xs2.ensure(static_cast<size_t>(std::max(R.n_scored, 1)) * d * 2);
  }
  if (k_ > 1 && fused_a2a()) plan_a2a_bytes();
  if (fused_a2a()) {  // this group's destinations of the fused all-to-all
    for (int p = 0; p < k_; ++p) h_peer_base_[p] = k_ == 1 ? ranks_[0].qkv.p : qh_dst(p);
    MRSP_CUDA(cudaMemcpyAsync(d_peer_base_, h_peer_base_.data(), 8 * sizeof(void*),
                              cudaMemcpyHostToDevice, s));
  }
}

// Bytes each local rank's fused exchanges send to OTHER ranks per layer,
// following the device routing exactly: the QKV epilogue's head-block routes
// (sequence -> heads) and the attention epilogue's O rows (heads -> sequence).
void Engine::plan_a2a_bytes() {
  const GroupState& g = grp_;
  const int nq = cfg_.n_q_heads, nkv = cfg_.n_kv_heads, nblk = nq + 2 * nkv;
  const int n_blocks = static_cast<int>((g.Ltot + ATTN_ROW_BLOCK - 1) / ATTN_ROW_BLOCK);
  a2a_fwd_bytes_.assign(ranks_.size(), 0);
  a2a_bwd_bytes_.assign(ranks_.size(), 0);
  auto owner = [&](long row) {  // sequence shard holding a token
    int p = 0;
    while (p + 1 < k_ && row >= token_b_[p + 1]) ++p;
    return p;
  };
  for (size_t i = 0; i < ranks_.size(); ++i) {
    const RankCtx& R = ranks_[i];
    for (int b = 0; b < n_blocks; ++b) {
      const long r0 = static_cast<long>(b) * ATTN_ROW_BLOCK, r1 = std::min(r0 + ATTN_ROW_BLOCK, g.Ltot);
      // forward: R's rows of this block, every head block to its owner(s)
      const long n = std::max(0L, std::min(r1, R.e) - std::max(r0, R.b));
      if (n > 0)
        for (int hb = 0; hb < nblk; ++hb) {
          const int2 d0 = route_h_[2 * hb], d1 = route_h_[2 * hb + 1];
          const int n_to = d1.x == -3 ? d1.y : d1.x == -2 ? 1 : 2;
          for (int t = 0; t < n_to; ++t) {
            const int dst = d1.x == -2 ? d0.x + attn_row_part(b, n_blocks, d1.y)
                          : d1.x == -3 ? d0.x + t : (t ? d1.x : d0.x);
            if (dst >= 0 && dst != R.g) a2a_fwd_bytes_[i] += static_cast<uint64_t>(n) * 256;
          }
        }
      // backward: O rows of the blocks R computes, to each token's shard
      if (R.hs.nq() == 0 ||
          (R.hs.rparts > 1 && attn_row_part(b, n_blocks, R.hs.rparts) != R.hs.rpart))
        continue;
      for (long r = r0; r < r1; ++r)
        if (owner(r) != R.g) a2a_bwd_bytes_[i] += static_cast<uint64_t>(R.hs.nq()) * 256;
    }
  }
}

// One model's pass over the packed group: pack, the decoder stack with Ulysses
// all-to-alls, final RMSNorm at the scored positions into R.xs / R.xs2.
void Engine::run_pass(const CacheEntry& emb, int model, int xs_slot) {
  const auto& c = cfg_;
  const GroupState& g = grp_;
  const LlmW& W = llm_[model];
  const int d = c.dim, nq = c.n_q_heads, nkv = c.n_kv_heads;
  const int Cqkv = (nq + 2 * nkv) * 128, Cq = nq * 128;
  cudaStream_t s = stream_;
  for (auto& R : ranks_) {
    Prof pm(*this, P_MISC);
    pack_sequence(emb.emb->as<bf16>(), static_cast<int>(g.n_frame_tok), g.d_question, g.n_q,
                  g.d_resp, g.d_len, g.Lmax, W.embed, d, R.b, static_cast<int>(R.e - R.b),
                  R.h.as<float>(), R.pos.as<int>(), R.pad.as<unsigned char>(), nullptr, s);
  }
  const float scale = 1.0f / std::sqrt(128.0f);
  int layer = -1;
  for (const auto& Lw : W.layers) {
    ++layer;
    for (size_t r = 0; r < stash_.size(); ++r) {  // backward: keep this layer's input
      const size_t nd = static_cast<size_t>(ranks_[r].e - ranks_[r].b) * d;
      if (nd)
        MRSP_CUDA(cudaMemcpyAsync(stash_[r] + layer * nd, ranks_[r].h.p, nd * 4,
                                  cudaMemcpyDeviceToDevice, s));
    }
    for (auto& R : ranks_) {
      const int n = static_cast<int>(R.e - R.b);
      if (n <= 0) continue;
      {
        Prof pm(*this, P_MISC);
        rmsnorm(R.h.as<float>(), d, Lw.attn_norm, R.xn.as<bf16>(), d, n, d, c.rms_eps, nullptr, s);
      }
      if (fused_a2a()) {
        // QKV projection + bias + RoPE + the Ulysses sequence -> head exchange
        // in one kernel: every head block lands in its owner rank's buffer
        Prof pg(*this, P_GEMM);
        GemmArgs ga{R.xn.p, Lw.wqkv, nullptr, n, Cqkv, d, d, d, 0, GEMM_EPI_QKV_SCATTER,
                    Lw.bqkv, nullptr, 0};
        ga.pos = R.pos.as<int>();
        ga.inv_freq = d_inv_freq_;
        ga.n_rope_blocks = nq + nkv;
        ga.row0 = k_ == 1 ? 0 : R.b;
        ga.route = d_route_;
        ga.peer_base = d_peer_base_;
        ga.peer_ld = d_peer_ld_;
        ga.row_blocks = static_cast<int>((g.Ltot + ATTN_ROW_BLOCK - 1) / ATTN_ROW_BLOCK);
        gemm_bf16(ga, s);
        if (k_ > 1) a2a_bytes.fetch_add(a2a_fwd_bytes_[&R - ranks_.data()]);
        continue;
      }
      {
        Prof pg(*this, P_GEMM);
        gemm_bf16({R.xn.p, Lw.wqkv, R.qkv.p, n, Cqkv, d, d, d, Cqkv, GEMM_EPI_BIAS_BF16, Lw.bqkv,
                   nullptr, 0},
                  s);
      }
      {
        Prof pm(*this, P_MISC);
        rope(R.qkv.as<bf16>(), Cqkv, 0, nq + nkv, R.pos.as<int>(), n, s);
      }
    }
    if (k_ > 1 && !fused_a2a()) a2a_forward(static_cast<int>(g.Ltot));
    if (mesh_) mesh_->barrier(s);  // every rank's head blocks have landed
    if (capture_kv_) {  // generation: keep this layer's prompt K and V of every
      // kv head, head-major [kv head][K | V][Lp][128] so decode streams
      // contiguous HBM. SP = 1: from the QKV rows; SP > 1: from the head shard
      // of a rank owning that kv head (a peer's landing buffer over NVLink) —
      // read before this layer's closing barrier, so before any rank's next
      // QKV scatter overwrites it.
      const size_t w = static_cast<size_t>(2 * nkv) * 128;
      bf16* dst = kv_prefix_.as<bf16>() + static_cast<size_t>(layer) * g.Lp * w;
      for (int j = 0; j < 2 * nkv; ++j) {  // j = 2 h + (0: K, 1: V)
        const int hkv = j >> 1, is_v = j & 1;
        const bf16* src;
        size_t ld;
        if (k_ == 1) {
          src = ranks_[0].qkv.as<bf16>() + static_cast<size_t>(nq + is_v * nkv + hkv) * 128;
          ld = Cqkv;
        } else {
          int p = 0;  // first rank holding kv head hkv (ranks without query heads get no K/V)
          while (!(split_of(p).kv_lo <= hkv && hkv < split_of(p).kv_hi && split_of(p).nq() > 0)) ++p;
          const HeadSplit hp = split_of(p);
          ld = static_cast<size_t>(hp.nq() + 2 * hp.nkv()) * 128;
          src = static_cast<const bf16*>(qh_dst(p)) +
                static_cast<size_t>(hp.nq() + is_v * hp.nkv() + (hkv - hp.kv_lo)) * 128;
        }
        MRSP_CUDA(cudaMemcpy2DAsync(dst + static_cast<size_t>(j) * g.Lp * 128, 256, src, ld * 2,
                                    256, g.Lp, cudaMemcpyDeviceToDevice, s));
      }
    }
    for (auto& R : ranks_) {
      const int nqr = R.hs.nq();
      if (nqr == 0) continue;
      Prof pa(*this, P_ATTN);
      const size_t ri = static_cast<size_t>(&R - ranks_.data());
      float* lse_keep = ri < stash_lse_.size()
                            ? stash_lse_[ri] + static_cast<size_t>(layer) * nqr * stash_lse_ld_
                            : nullptr;
      if (k_ == 1) {
        AttnParams ap{R.qkv.p, Cqkv, 0, R.qkv.p, Cqkv, nq * 128, R.qkv.p, Cqkv, (nq + nkv) * 128,
                      R.ol.p, Cq, 0, static_cast<int>(g.Ltot), nq, nq / nkv, scale,
                      ATTN_CAUSAL_PREFIX, static_cast<int>(g.Lp), g.Lmax, 0};
        ap.lse = lse_keep;
        ap.lse_ld = stash_lse_ld_;
        attention_fwd(ap, s);
      } else {
        const int Cr = (nqr + 2 * R.hs.nkv()) * 128;
        void* qh = fused_a2a() ? qh_dst(R.g) : R.qh.p;
        AttnParams ap{qh, Cr, 0, qh, Cr, nqr * 128, qh, Cr,
                      (nqr + R.hs.nkv()) * 128, R.oh.p, nqr * 128, 0, static_cast<int>(g.Ltot),
                      nqr, R.hs.q_per_kv, scale, ATTN_CAUSAL_PREFIX, static_cast<int>(g.Lp),
                      g.Lmax, 0};
        if (fused_a2a()) {
          // the head -> sequence exchange in the attention epilogue: each O
          // row goes straight to the rank owning that token
          ap.n_dst = k_;
          for (int p = 0; p < k_; ++p) {
            ap.dst_bounds[p] = token_b_[p];
            ap.dst_base[p] = ol_dst(p);
          }
          a2a_bytes.fetch_add(a2a_bwd_bytes_[&R - ranks_.data()]);
          ap.row_parts = R.hs.rparts;
          ap.row_part = R.hs.rpart;
          ap.dst_bounds[k_] = token_e_[k_ - 1];
          ap.dst_ld = Cq;
          ap.dst_col0 = R.hs.q_lo * 128;
        }
        ap.lse = lse_keep;
        ap.lse_ld = stash_lse_ld_;
        attention_fwd(ap, s);
      }
    }
    if (k_ > 1 && !fused_a2a()) a2a_backward(static_cast<int>(g.Ltot));
    if (mesh_) mesh_->barrier(s);  // every rank's O rows have landed
    for (size_t r = 0; r < stash_o_.size(); ++r) {  // backward: keep this layer's O
      const size_t nc = static_cast<size_t>(ranks_[r].e - ranks_[r].b) * Cq;
      if (nc)
        MRSP_CUDA(cudaMemcpyAsync(stash_o_[r] + layer * nc, mesh_ ? ol_dst(ranks_[r].g) : ranks_[r].ol.p,
                                  nc * 2, cudaMemcpyDeviceToDevice, s));
    }
    for (auto& R : ranks_) {
      const int n = static_cast<int>(R.e - R.b);
      if (n <= 0) continue;
      {
        Prof pg(*this, P_GEMM);
        gemm_bf16({mesh_ ? ol_dst(R.g) : R.ol.p, Lw.wo, nullptr, n, d, Cq, Cq, Cq, 0,
                   GEMM_EPI_RESID_F32, nullptr, R.h.as<float>(), d},
                  s);
      }
      {
        Prof pm(*this, P_MISC);
        rmsnorm(R.h.as<float>(), d, Lw.mlp_norm, R.xn.as<bf16>(), d, n, d, c.rms_eps, nullptr, s);
      }
      {
        Prof pg(*this, P_GEMM);
        gemm_bf16({R.xn.p, Lw.wgu, R.act.p, n, 2 * c.mlp, d, d, d, c.mlp, GEMM_EPI_SWIGLU_BF16,
                   nullptr, nullptr, 0},
                  s);
        gemm_bf16({R.act.p, Lw.wdown, nullptr, n, d, c.mlp, c.mlp, c.mlp, 0, GEMM_EPI_RESID_F32,
                   nullptr, R.h.as<float>(), d},
                  s);
      }
    }
  }
  for (auto& R : ranks_) {
    if (R.n_scored == 0) continue;
    DevBuf& xs = xs_slot ? R.xs2 : R.xs;
    rmsnorm(R.h.as<float>(), d, W.final_norm, xs.as<bf16>(), d, R.n_scored, d, c.rms_eps,
            R.scored_idx.as<int32_t>(), s);
  }
}

namespace {
__global__ void scatter3_kernel(const float* __restrict__ src, const int* __restrict__ slot, int n,
                                int nvec, float* __restrict__ dst, long stride) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n)
    for (int v = 0; v < nvec; ++v) dst[v * stride + slot[i]] = src[v * n + i];
}
}  // namespace

// Scatter per-shard vectors into the group-ordered outputs, reduce across
// processes, copy out.
void Engine::finish_group(int nvec, float* const* outs, bool out_on_device) {
  const GroupState& g = grp_;
  cudaStream_t s = stream_;
  if (mesh_) {
    // each rank writes its scored positions into every rank's landing buffer
    const long stride = mesh_->caps().scored + 16;
    const RankCtx& R = ranks_[0];
    Prof pc(*this, P_COMM);
    mesh_->barrier(s);  // every rank has read the previous group's outputs
    if (R.lm_n)
      for (int p = 0; p < k_; ++p) {
        scatter3_kernel<<<(R.lm_n + 255) / 256, 256, 0, s>>>(
            R.lp.as<float>(), R.lm_idx.as<int32_t>() + R.lm_n, R.lm_n, nvec, mesh_->lp(p), stride);
        count_launch();
        MRSP_CUDA(cudaGetLastError());
      }
    mesh_->barrier(s);
    const cudaMemcpyKind kind = out_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    for (int v = 0; v < nvec; ++v)
      if (outs[v] && g.total_scored)
        MRSP_CUDA(cudaMemcpyAsync(outs[v], mesh_->lp(R.g) + v * stride, g.total_scored * 4, kind, s));
    MRSP_CUDA(cudaStreamSynchronize(s));
    prof_collect();
    return;
  }
  for (auto& R : ranks_) {
    if (R.lm_n == 0) continue;
    scatter3_kernel<<<(R.lm_n + 255) / 256, 256, 0, s>>>(
        R.lp.as<float>(), R.lm_idx.as<int32_t>() + R.lm_n, R.lm_n, nvec, g.full, g.stride);
    count_launch();
    MRSP_CUDA(cudaGetLastError());
  }
  if (nccl_) {
    Prof pc(*this, P_COMM);
    nccl_->all_reduce_sum_f32(g.full, g.full, static_cast<size_t>(nvec * g.stride), s);
  }
  const cudaMemcpyKind kind = out_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  for (int v = 0; v < nvec; ++v)
    if (outs[v] && g.total_scored)
      MRSP_CUDA(cudaMemcpyAsync(outs[v], g.full + v * g.stride, g.total_scored * 4, kind, s));
  MRSP_CUDA(cudaStreamSynchronize(s));
  prof_collect();
}

const void* Engine::lm_rows(RankCtx& R, int m) {
  if (!spread_lm()) return (m ? R.xs2 : R.xs).p;
  const size_t cap = mesh_ ? static_cast<size_t>(mesh_->caps().lm_rows) : static_cast<size_t>(R.lm_n);
  const void* base = mesh_ ? mesh_->xs(R.g) : R.lmx.p;
  return static_cast<const bf16*>(base) + static_cast<size_t>(m) * cap * cfg_.dim;
}

// Spread LM head: every owner copies its scored tokens' final-norm rows into
// the landing rows of the rank(s) whose LM-head slice holds them (copy-engine
// P2P over NVLink between processes; a device copy between virtual ranks).
void Engine::lm_exchange(int n_models) {
  if (!spread_lm()) return;
  const GroupState& g = grp_;
  const int d = cfg_.dim;
  const auto lm_plan = plan(g.total_scored, k_);
  Prof pc(*this, P_COMM);
  if (mesh_) mesh_->barrier(stream_);  // every rank has consumed its previous slice
  for (auto& R : ranks_) {
    for (int p = 0; p < k_; ++p) {
      const long lo = std::max<long>(R.sc_lo, static_cast<long>(lm_plan[p].first));
      const long hi = std::min<long>(R.sc_lo + R.n_scored, static_cast<long>(lm_plan[p].second));
      if (hi <= lo) continue;
      const size_t cap = mesh_ ? static_cast<size_t>(mesh_->caps().lm_rows)
                               : static_cast<size_t>(ranks_[p].lm_n);
      bf16* dst = static_cast<bf16*>(mesh_ ? mesh_->xs(p) : ranks_[p].lmx.p);
      for (int m = 0; m < n_models; ++m) {
        const bf16* src = (m ? R.xs2 : R.xs).as<bf16>();
        MRSP_CUDA(cudaMemcpyAsync(dst + (m * cap + (lo - static_cast<long>(lm_plan[p].first))) * d,
                                  src + static_cast<size_t>(lo - R.sc_lo) * d,
                                  static_cast<size_t>(hi - lo) * d * 2, cudaMemcpyDeviceToDevice,
                                  stream_));
      }
      if (p != R.g) a2a_bytes.fetch_add(static_cast<uint64_t>(hi - lo) * d * 2 * n_models);
    }
  }
  if (mesh_) mesh_->barrier(stream_);  // every slice has landed
}

void Engine::prefill_logprobs(const CacheEntry& emb, const int32_t* question, int n_q,
                              const int32_t* resp, const int32_t* lengths, int G, int Lmax,
                              int model, float* lp_out, float* lse_out, bool out_on_device) {
  MRSP_REQUIRE(model == 0 || model == 1, MRSP_INVALID_ARGUMENT, "prefill: model must be 0 or 1");
  std::lock_guard<std::mutex> run(run_mu_);
  prepare_group(emb, question, n_q, resp, lengths, G, Lmax);
  run_pass(emb, model, 0);
  lm_exchange(1);
  const auto& c = cfg_;
  for (auto& R : ranks_) {
    const int ns = R.lm_n;
    if (ns == 0) continue;
    float* lp = static_cast<float*>(R.lp.ensure(static_cast<size_t>(ns) * 4 * 3));
    const size_t wsb = lmhead_workspace_bytes(ns, c.vocab);
    void* ws = R.ws.ensure(wsb);
    Prof pl(*this, P_LMHEAD);
    lmhead_logprob(lm_rows(R, 0), c.dim, llm_[model].lm_head, ns, c.vocab, c.dim,
                   R.lm_idx.as<int32_t>(), lp, lp + ns, ws, wsb, stream_);
  }
  float* outs[2] = {lp_out, lse_out};
  finish_group(2, outs, out_on_device);
}

// Both passes + the fused dual LM head: per-token log pi_theta(y), log pi_ref(y)
// and exact KL(pi_theta || pi_ref) from one vocabulary sweep.
void Engine::group_logprobs(const CacheEntry& emb, const int32_t* question, int n_q,
                            const int32_t* resp, const int32_t* lengths, int G, int Lmax,
                            float* lp_policy, float* lp_ref, float* kl, bool out_on_device) {
  std::lock_guard<std::mutex> run(run_mu_);
  prepare_group(emb, question, n_q, resp, lengths, G, Lmax);
  run_pass(emb, 0, 0);
  run_pass(emb, 1, 1);
  lm_exchange(2);
  const auto& c = cfg_;
  for (auto& R : ranks_) {
    const int ns = R.lm_n;
    if (ns == 0) continue;
    float* lp = static_cast<float*>(R.lp.ensure(static_cast<size_t>(ns) * 4 * 3));
    const size_t wsb = lmhead_dual_workspace_bytes(ns, c.vocab);
    void* ws = R.ws.ensure(wsb);
    Prof pl(*this, P_LMHEAD);
    lmhead_dual_logprob_kl(lm_rows(R, 0), llm_[0].lm_head, lm_rows(R, 1), llm_[1].lm_head, ns,
                           c.vocab, c.dim, R.lm_idx.as<int32_t>(), lp, lp + ns, lp + 2 * ns, ws,
                           wsb, stream_);
  }
  float* outs[3] = {lp_policy, lp_ref, kl};
  finish_group(3, outs, out_on_device);
}

void Engine::generate(const CacheEntry& emb, const int32_t* question, int n_q, int G,
                      int max_len, float temperature, uint64_t seed, int32_t* tokens_out,
                      int32_t* lengths_out, float* old_lp_out) {
  const auto& c = cfg_;
  // SP > 1: the prompt prefill is sequence-parallel and every rank gathers the
  // prompt K/V of all kv heads from the head shards; the G-row decode then runs
  // on every rank (replicated: bit-identical tokens and log-probs everywhere).
  MRSP_REQUIRE(!nccl_, MRSP_INVALID_ARGUMENT,
               "generate: SP > 1 needs the peer-memory transport (no NCCL id)");
  MRSP_REQUIRE(temperature > 0.f, MRSP_INVALID_ARGUMENT,
               "sample_rollout: temperature must be > 0");
  MRSP_REQUIRE(max_len >= 1, MRSP_INVALID_ARGUMENT, "sample_rollout: max_len must be >= 1");
  const int nq = c.n_q_heads, nkv = c.n_kv_heads, qpk = nq / nkv, d = c.dim;
  MRSP_REQUIRE(G >= 1 && G * qpk <= 64, MRSP_INVALID_ARGUMENT,
               "generate: 1 <= G and G x q_per_kv <= 64");
  std::lock_guard<std::mutex> run(run_mu_);
  cudaStream_t s = stream_;
  // 1. prompt prefill (the policy over [video | question]) keeping every layer's K/V
  const int32_t dummy_resp = 0, zero_len = 0;
  prepare_group(emb, question, n_q, &dummy_resp, &zero_len, 1, 1);
  const long Lp = grp_.Lp;
  const size_t kvw = static_cast<size_t>(2 * nkv) * 128;  // one position's K | V
  kv_prefix_.ensure(static_cast<size_t>(c.layers) * std::max<long>(Lp, 1) * kvw * 2);
  capture_kv_ = true;
  try {
    run_pass(emb, 0, 0);
  } catch (...) {
    capture_kv_ = false;
    throw;
  }
  capture_kv_ = false;
  // 2. decode state
  const int Cqkv = (nq + 2 * nkv) * 128, Cq = nq * 128;
  RankCtx& R = ranks_[0];
  DevBuf& st = R.recv;  // generation scratch (R.send/R.recv serve only the NCCL exchange)
  const size_t n_tok = static_cast<size_t>(G) * max_len;
  size_t off = 0;
  auto carve = [&](size_t bytes) {
    const size_t o = off;
    off = (off + bytes + 255) & ~size_t(255);
    return o;
  };
  const size_t o_rows = carve(static_cast<size_t>(c.layers) * max_len * G * kvw * 2);
  const size_t o_h = carve(static_cast<size_t>(G) * d * 4), o_xn = carve(static_cast<size_t>(G) * d * 2);
  const size_t o_qkv = carve(static_cast<size_t>(G) * Cqkv * 2), o_o = carve(static_cast<size_t>(G) * Cq * 2);
  const size_t o_act = carve(static_cast<size_t>(G) * c.mlp * 2);
  const size_t o_logit = carve(static_cast<size_t>(G) * c.vocab * 4);
  const size_t o_part = carve(decode_partial_bytes(static_cast<int>(Lp), max_len, G, nkv));
  const size_t o_tok = carve(n_tok * 4), o_lp = carve(n_tok * 4), o_len = carve(G * 4);
  const size_t o_done = carve(G * 4), o_pos = carve(G * 4), o_t = carve(4);
  const size_t splitk_bytes = gemm_splitk_ws_bytes(G), o_splitk = carve(splitk_bytes);
  const size_t o_sample = carve(sample_workspace_bytes(G));
  uint8_t* b = static_cast<uint8_t*>(st.ensure(off));
  bf16* kv_rows = reinterpret_cast<bf16*>(b + o_rows);
  float* h = reinterpret_cast<float*>(b + o_h);
  bf16* xn = reinterpret_cast<bf16*>(b + o_xn);
  bf16* qkv = reinterpret_cast<bf16*>(b + o_qkv);
  bf16* od = reinterpret_cast<bf16*>(b + o_o);
  bf16* act = reinterpret_cast<bf16*>(b + o_act);
  float* logits = reinterpret_cast<float*>(b + o_logit);
  float* part = reinterpret_cast<float*>(b + o_part);
  int* tokens = reinterpret_cast<int*>(b + o_tok);
  float* old_lp = reinterpret_cast<float*>(b + o_lp);
  int* lengths = reinterpret_cast<int*>(b + o_len);
  int* done = reinterpret_cast<int*>(b + o_done);
  int* pos = reinterpret_cast<int*>(b + o_pos);
  int* tdev = reinterpret_cast<int*>(b + o_t);  // the step index t, advanced on the device
  // G-row GEMMs split K over the SMs (MRSP_DECODE_SPLITK=0: one CTA per n tile)
  const char* env_sk = std::getenv("MRSP_DECODE_SPLITK");
  float* splitk = (env_sk && std::atoi(env_sk) == 0) ? nullptr
                                                     : reinterpret_cast<float*>(b + o_splitk);
  auto dec_gemm = [&](GemmArgs g) {
    g.splitk_ws = splitk;
    g.splitk_ws_bytes = splitk_bytes;
    gemm_bf16(g, s);
  };
  MRSP_CUDA(cudaMemsetAsync(kv_rows, 0, static_cast<size_t>(c.layers) * max_len * G * kvw * 2, s));
  // TMA descriptors of every layer's prompt K/V and row cache, built once
  const bool tc_decode = decode_use_tensor_cores(static_cast<int>(Lp));
  std::vector<CUtensorMap> maps(tc_decode ? 2 * c.layers : 0);
  for (int l = 0; tc_decode && l < c.layers; ++l)
    decode_tensor_maps(kv_prefix_.as<bf16>() + static_cast<size_t>(l) * Lp * kvw, static_cast<int>(Lp),
                       nkv, kv_rows + static_cast<size_t>(l) * max_len * G * kvw,
                       static_cast<long>(max_len) * G, static_cast<int>(kvw), &maps[2 * l]);
  MRSP_CUDA(cudaMemsetAsync(tokens, 0, n_tok * 4, s));  // PAD
  MRSP_CUDA(cudaMemsetAsync(old_lp, 0, n_tok * 4, s));
  MRSP_CUDA(cudaMemsetAsync(lengths, 0, G * 4, s));
  MRSP_CUDA(cudaMemsetAsync(done, 0, G * 4, s));
  MRSP_CUDA(cudaMemsetAsync(tdev, 0, 4, s));
  const LlmW& W = llm_[0];
  const float scale = 1.0f / std::sqrt(128.0f);
  std::vector<int> done_h(G);
  // 3. one decode step: tokens -> embeddings -> 28 layers (G-row GEMMs, decode
  // attention over prompt K/V + own-row K/V) -> LM head logits -> sample -> t + 1.
  // Every kernel reads t from `tdev`; t_grid only sizes the attention grid.
  // Decode fusions (MRSP_DECODE_FUSE=0: off): the first RMSNorm rides on the
  // token embedding, RoPE + the K|V row-cache append on the QKV split-K
  // reduction, and each following RMSNorm on the residual split-K reduction
  // before it (O projection -> MLP norm, down projection -> next layer's
  // attention norm or the final norm). Same bits as the separate kernels.
  const char* env_fuse = std::getenv("MRSP_DECODE_FUSE");
  const bool fuse = !(env_fuse && std::atoi(env_fuse) == 0);
  auto step = [&](int t_grid) {
    bool xn_ready = false;  // xn already holds the norm the next GEMM needs
    {
      Prof pm(*this, P_MISC);
      decode_embed(W.embed, d, tokens, max_len, tdev, G, static_cast<int>(Lp), h, pos, s,
                   fuse ? W.layers[0].attn_norm : nullptr, xn, c.rms_eps);
      xn_ready = fuse;
    }
    for (int l = 0; l < c.layers; ++l) {
      const LlmLayerW& Lw = W.layers[l];
      const float* next_norm = l + 1 < c.layers ? W.layers[l + 1].attn_norm : W.final_norm;
      if (!xn_ready) {
        Prof pm(*this, P_MISC);
        rmsnorm(h, d, Lw.attn_norm, xn, d, G, d, c.rms_eps, nullptr, s);
      }
      bf16* rows_l = kv_rows + static_cast<size_t>(l) * max_len * G * kvw;
      bool roped = false;
      {
        Prof pg(*this, P_GEMM);
        GemmArgs ga{xn, Lw.wqkv, qkv, G, Cqkv, d, d, d, Cqkv, GEMM_EPI_BIAS_BF16, Lw.bqkv, nullptr, 0};
        if (fuse) {
          ga.post = GEMM_POST_ROPE_APPEND;
          ga.pos = pos;
          ga.inv_freq = d_inv_freq_;
          ga.n_rope_blocks = nq + nkv;
          ga.kv_rows = rows_l;
          ga.kvw = static_cast<int>(kvw);
          ga.kv_col0 = nq * 128;
          ga.tdev = tdev;
        }
        ga.splitk_ws = splitk;
        ga.splitk_ws_bytes = splitk_bytes;
        roped = gemm_bf16(ga, s);
      }
      if (!roped) {
        Prof pm(*this, P_MISC);
        rope(qkv, Cqkv, 0, nq + nkv, pos, G, s);
        decode_append_kv(qkv, Cqkv, nq * 128, rows_l, static_cast<int>(kvw), G, tdev, s);
      }
      {
        Prof pa(*this, P_ATTN);
        decode_attention(qkv, Cqkv, 0, kv_prefix_.as<bf16>() + static_cast<size_t>(l) * Lp * kvw,
                         rows_l, static_cast<int>(kvw), nkv * 128, static_cast<int>(Lp), G, t_grid,
                         max_len * G, tdev, qpk, nkv, scale, part, od, Cq, s,
                         tc_decode ? &maps[2 * l] : nullptr);
      }
      // residual GEMM (h += A W^T), optionally followed by the fused norm -> xn
      auto resid_gemm = [&](const bf16* A, const bf16* Wt, int K, const float* norm_w) {
        Prof pg(*this, P_GEMM);
        GemmArgs ga{A, Wt, nullptr, G, d, K, K, K, 0, GEMM_EPI_RESID_F32, nullptr, h, d};
        if (fuse) {
          ga.post = GEMM_POST_RMSNORM;
          ga.norm_w = norm_w;
          ga.norm_out = xn;
          ga.ld_norm = d;
          ga.norm_eps = c.rms_eps;
        }
        ga.splitk_ws = splitk;
        ga.splitk_ws_bytes = splitk_bytes;
        return gemm_bf16(ga, s);
      };
      xn_ready = resid_gemm(od, Lw.wo, Cq, Lw.mlp_norm);
      if (!xn_ready) {
        Prof pm(*this, P_MISC);
        rmsnorm(h, d, Lw.mlp_norm, xn, d, G, d, c.rms_eps, nullptr, s);
      }
      {
        Prof pg(*this, P_GEMM);
        dec_gemm({xn, Lw.wgu, act, G, 2 * c.mlp, d, d, d, c.mlp, GEMM_EPI_SWIGLU_BF16, nullptr,
                  nullptr, 0});
      }
      xn_ready = resid_gemm(act, Lw.wdown, c.mlp, next_norm);
    }
    {
      Prof pl(*this, P_LMHEAD);
      if (!xn_ready) rmsnorm(h, d, W.final_norm, xn, d, G, d, c.rms_eps, nullptr, s);
      dec_gemm({xn, W.lm_head, logits, G, c.vocab, d, d, d, c.vocab, GEMM_EPI_STORE_F32, nullptr,
                nullptr, 0});
    }
    {
      Prof psm(*this, P_MISC);
      sample_tokens(logits, G, c.vocab, temperature, seed, tdev, done, tokens, old_lp, lengths,
                    max_len, b + o_sample, s);
      decode_step_advance(tdev, s);
    }
  };
  // Steps t >= 1 replay one CUDA graph of a step, captured with the attention
  // grid sized for t = max_len - 1: the ~13 launches per layer become one graph
  // launch per step. Step 0 runs eagerly (one-time kernel attribute setup).
  // MRSP_DECODE_GRAPH=0 launches every step eagerly; the CUDA-core decode
  // attention (MRSP_DECODE_CC=1) is eager only.
  const char* env_graph = std::getenv("MRSP_DECODE_GRAPH");
  const bool use_graph = tc_decode && max_len > 2 && !(env_graph && std::atoi(env_graph) == 0);
  // MRSP_DECODE_PDL=1: programmatic dependent launches inside the graph (each
  // kernel's launch and prologue overlap its predecessor's tail). Measured
  // neutral at c4 and 15-25% slower at c2 (profiles/r1_generation_perf.jsonl),
  // so off by default.
  const char* env_pdl = std::getenv("MRSP_DECODE_PDL");
  const bool use_pdl = env_pdl && std::atoi(env_pdl) != 0;
  struct GraphGuard {
    cudaGraph_t g = nullptr;
    cudaGraphExec_t x = nullptr;
    ~GraphGuard() {
      if (x) cudaGraphExecDestroy(x);
      if (g) cudaGraphDestroy(g);
    }
  } graph;
  uint64_t graph_launches = 0;
  for (int t = 0; t < max_len; ++t) {
    if (!use_graph || t == 0) {
      step(t);
    } else {
      if (!graph.x) {
        const bool prof_was = prof_;
        prof_ = false;  // no timing events inside the capture
        const uint64_t n0 = mrsp_launch_count();
        MRSP_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        try {
          PdlScope pdl(use_pdl);
          step(max_len - 1);
        } catch (...) {
          cudaGraph_t dead = nullptr;
          cudaStreamEndCapture(s, &dead);
          if (dead) cudaGraphDestroy(dead);
          prof_ = prof_was;
          throw;
        }
        MRSP_CUDA(cudaStreamEndCapture(s, &graph.g));
        prof_ = prof_was;
        graph_launches = mrsp_launch_count() - n0;
        MRSP_CUDA(cudaGraphInstantiate(&graph.x, graph.g, 0));
      }
      Prof pd(*this, P_DECODE_GRAPH);
      MRSP_CUDA(cudaGraphLaunch(graph.x, s));
      count_launch(graph_launches);
    }
    if ((t & 15) == 15 || t == max_len - 1) {  // stop once every row has sampled EOS
      MRSP_CUDA(cudaMemcpyAsync(done_h.data(), done, G * 4, cudaMemcpyDeviceToHost, s));
      MRSP_CUDA(cudaStreamSynchronize(s));
      bool all = true;
      for (int v : done_h) all = all && v;
      if (all) break;
    }
  }
  MRSP_CUDA(cudaMemcpyAsync(tokens_out, tokens, n_tok * 4, cudaMemcpyDeviceToHost, s));
  MRSP_CUDA(cudaMemcpyAsync(old_lp_out, old_lp, n_tok * 4, cudaMemcpyDeviceToHost, s));
  MRSP_CUDA(cudaMemcpyAsync(lengths_out, lengths, G * 4, cudaMemcpyDeviceToHost, s));
  MRSP_CUDA(cudaStreamSynchronize(s));
  prof_collect();
}

size_t Engine::p2p_export(int max_frames, long max_tokens, long max_scored, void* blob) {
  MRSP_REQUIRE(mesh_ != nullptr, MRSP_LOGIC_ERROR, "p2p: engine was created with NCCL or 1 process");
  MRSP_REQUIRE(max_frames >= 1 && max_tokens >= 1 && max_scored >= 0, MRSP_INVALID_ARGUMENT,
               "p2p: capacities must be positive");
  const RankCtx& R = ranks_[0];
  PeerCaps caps;
  caps.tokens = max_tokens;
  caps.shard = (max_tokens + k_ - 1) / k_;
  caps.frames = max_frames;
  caps.scored = max_scored;
  caps.c_head_shard = std::max(1, R.hs.nq() + 2 * R.hs.nkv()) * 128;
  caps.cq = cfg_.n_q_heads * 128;
  caps.tok_row = tokens_per_frame() * cfg_.dim;
  caps.lm_rows = (max_scored + k_ - 1) / k_;
  caps.dim = cfg_.dim;
  caps.cq_me = std::max(1, R.hs.nq()) * 128;
  caps.cqkv = (cfg_.n_q_heads + 2 * cfg_.n_kv_heads) * 128;
  caps.red_floats = kGradReduceChunk;
  caps.m_kv = k_ > cfg_.n_kv_heads ? k_ / cfg_.n_kv_heads : 1;
  caps.nkv = cfg_.n_kv_heads;
  if (blob) mesh_->export_blob(caps, blob);
  return PeerMesh::kBlobBytes;
}

void Engine::p2p_import(const void* blobs) {
  MRSP_REQUIRE(mesh_ != nullptr, MRSP_LOGIC_ERROR, "p2p: engine was created with NCCL or 1 process");
  mesh_->import_blobs(blobs);
}

size_t Engine::cache_size() {
  std::lock_guard<std::mutex> lock(cache_mu_);
  return cache_.size();
}
void Engine::cache_clear() {
  std::lock_guard<std::mutex> lock(cache_mu_);
  cache_.clear();
}
// ---------------------------------------------------------------------------
// Embedding-cache persistence (the reference never persists
// its cache, engine.hpp:105-128). File: "MRSPEMB1", u32 version 1, frames,
// tokens/frame, dim, dtype (1 = bf16), u64 fingerprint of the vision + projector
// geometry, then [frames * tokens][dim] bf16 row-major.
namespace {
constexpr char kEmbMagic[8] = {'M', 'R', 'S', 'P', 'E', 'M', 'B', '1'};
struct EmbHeader {
  char magic[8];
  uint32_t version, frames, tokens, dim, dtype, pad;
  uint64_t fingerprint;
};
static_assert(sizeof(EmbHeader) == 40, "packed header");
uint64_t encoder_fingerprint(const mrsp_model_config& c) {
  const int v[] = {c.image_size, c.patch, c.v_dim, c.v_heads, c.v_head_dim, c.v_mlp, c.v_layers,
                   c.dim};
  std::string s;
  for (int x : v) s += std::to_string(x) + ",";
  return fnv1a(s);
}
}  // namespace

void Engine::cache_save(const CacheEntry& e, const std::string& path) {
  const int T = tokens_per_frame();
  const size_t n = static_cast<size_t>(e.n_frames) * T * cfg_.dim;
  std::vector<uint16_t> host(n);
  MRSP_CUDA(cudaMemcpy(host.data(), e.emb->p, n * 2, cudaMemcpyDeviceToHost));
  EmbHeader h{};
  std::memcpy(h.magic, kEmbMagic, 8);
  h.version = 1;
  h.frames = static_cast<uint32_t>(e.n_frames);
  h.tokens = static_cast<uint32_t>(T);
  h.dim = static_cast<uint32_t>(cfg_.dim);
  h.dtype = 1;
  h.fingerprint = encoder_fingerprint(cfg_);
  FILE* f = std::fopen(path.c_str(), "wb");
  MRSP_REQUIRE(f != nullptr, MRSP_RUNTIME_ERROR, "cache_save: cannot open " + path);
  const bool ok = std::fwrite(&h, sizeof(h), 1, f) == 1 && std::fwrite(host.data(), 2, n, f) == n;
  const bool closed = std::fclose(f) == 0;
  MRSP_REQUIRE(ok && closed, MRSP_RUNTIME_ERROR, "cache_save: write failed: " + path);
}

std::shared_ptr<CacheEntry> Engine::cache_load(const std::string& id, const std::string& path) {
  FILE* f = std::fopen(path.c_str(), "rb");
  MRSP_REQUIRE(f != nullptr, MRSP_RUNTIME_ERROR, "cache_load: cannot open " + path);
  EmbHeader h{};
  const bool got = std::fread(&h, sizeof(h), 1, f) == 1;
  if (!got || std::memcmp(h.magic, kEmbMagic, 8) != 0 || h.version != 1 || h.dtype != 1) {
    std::fclose(f);
    fail(MRSP_INVALID_ARGUMENT, "cache_load: not an MRSP embedding file: " + path);
  }
  if (static_cast<int>(h.tokens) != tokens_per_frame() || static_cast<int>(h.dim) != cfg_.dim ||
      h.fingerprint != encoder_fingerprint(cfg_) || h.frames < 1) {
    std::fclose(f);
    fail(MRSP_INVALID_ARGUMENT, "cache_load: embeddings were made by a different encoder geometry");
  }
  const size_t n = static_cast<size_t>(h.frames) * h.tokens * h.dim;
  std::vector<uint16_t> host(n);
  const bool read_ok = std::fread(host.data(), 2, n, f) == n;
  std::fclose(f);
  MRSP_REQUIRE(read_ok, MRSP_RUNTIME_ERROR, "cache_load: truncated file " + path);
  auto emb = std::make_shared<DevBuf>();
  MRSP_CUDA(cudaMemcpy(emb->ensure(n * 2), host.data(), n * 2, cudaMemcpyHostToDevice));
  auto entry = std::make_shared<CacheEntry>();
  entry->emb = emb;
  entry->n_frames = static_cast<int>(h.frames);
  entry->ready = true;
  std::lock_guard<std::mutex> lock(cache_mu_);
  entry->seq = ++cache_seq_;
  cache_[id] = entry;  // later fetches of `id` hit without encoding
  if (cache_capacity > 0)
    while (static_cast<int>(cache_.size()) > cache_capacity) {
      auto oldest = std::min_element(cache_.begin(), cache_.end(), [](auto& a, auto& b) {
        return a.second->seq < b.second->seq;
      });
      cache_.erase(oldest);
    }
  return entry;
}

size_t Engine::embedding_bytes(const CacheEntry& e) const {
  return static_cast<size_t>(e.n_frames) * tokens_per_frame() * cfg_.dim * 2;
}

void Engine::copy_embeddings(const CacheEntry& e, void* host_out) {
  MRSP_CUDA(cudaMemcpy(host_out, e.emb->p, embedding_bytes(e), cudaMemcpyDeviceToHost));
}

}  // namespace mrsp

// ============================================================================
// C-ABI
// ============================================================================
struct mrsp_engine {
  std::unique_ptr<mrsp::Engine> impl;
  std::mutex mu;
  std::map<std::string, std::shared_ptr<mrsp::CacheEntry>> last;  // pins for prefill
};

using namespace mrsp;

extern "C" mrsp_status mrsp_ulysses_plan(int n_q, int n_kv, int sp, int rank, int32_t* out14) {
  return guard([&] {
    MRSP_REQUIRE(sp >= 1 && rank >= 0 && rank < sp, MRSP_INVALID_ARGUMENT, "ulysses: bad rank");
    const HeadSplit hs = head_split(n_q, n_kv, sp, rank);
    out14[0] = hs.q_lo;
    out14[1] = hs.q_hi;
    out14[2] = hs.kv_lo;
    out14[3] = hs.kv_hi;
    out14[4] = hs.q_per_kv;
    const auto b = ulysses_blocks(n_q, n_kv, hs);
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) out14[5 + 3 * i + j] = b[i][j];
  });
}

extern "C" mrsp_status mrsp_head_split(int n_q, int n_kv, int sp, int rank, int row_split,
                                       int32_t* out7) {
  return guard([&] {
    MRSP_REQUIRE(sp >= 1 && rank >= 0 && rank < sp && out7, MRSP_INVALID_ARGUMENT,
                 "ulysses: bad rank");
    const HeadSplit hs = head_split(n_q, n_kv, sp, rank, row_split != 0);
    const int32_t v[7] = {hs.q_lo, hs.q_hi, hs.kv_lo, hs.kv_hi, hs.q_per_kv, hs.rparts, hs.rpart};
    std::memcpy(out7, v, sizeof(v));
  });
}

extern "C" int mrsp_attn_row_part(int block, int n_blocks, int m) {
  if (m < 1 || n_blocks < 1 || block < 0 || block >= n_blocks) return -1;
  return mrsp::attn_row_part(block, n_blocks, m);
}

extern "C" size_t mrsp_p2p_blob_bytes(void) { return mrsp::PeerMesh::kBlobBytes; }

extern "C" mrsp_status mrsp_nccl_unique_id(void* out128) {
  return guard([&] { Nccl::unique_id(out128); });
}

extern "C" mrsp_status mrsp_engine_create(const mrsp_model_config* cfg, int sp_degree,
                                          int proc_rank, int n_procs, uint64_t vision_seed,
                                          uint64_t policy_seed, uint64_t ref_seed, int with_ref,
                                          const void* nccl_id, mrsp_engine** out) {
  return guard([&] {
    MRSP_REQUIRE(cfg && out, MRSP_INVALID_ARGUMENT, "engine: null argument");
    auto e = std::make_unique<mrsp_engine>();
    e->impl = std::make_unique<Engine>(*cfg, sp_degree, proc_rank, n_procs, vision_seed,
                                       policy_seed, ref_seed, with_ref, nccl_id);
    *out = e.release();
  });
}

extern "C" mrsp_status mrsp_engine_destroy(mrsp_engine* e) {
  return guard([&] { delete e; });
}

static std::shared_ptr<CacheEntry> lookup(mrsp_engine* e, const char* id) {
  std::lock_guard<std::mutex> lock(e->mu);
  auto it = e->last.find(id);
  MRSP_REQUIRE(it != e->last.end(), MRSP_INVALID_ARGUMENT,
               std::string("prefill: video not encoded: ") + id);
  return it->second;
}

// The entries the last encodes / steps produced, by video id (<= 4 kept): what
// prefill and get_embeddings resolve a video id to, also for cache-off fills.
static void remember(mrsp_engine* e, const char* video_id, const std::shared_ptr<CacheEntry>& entry) {
  std::lock_guard<std::mutex> lock(e->mu);
  e->last[video_id] = entry;
  while (e->last.size() > 4) {
    auto oldest = std::min_element(e->last.begin(), e->last.end(),
                                   [](auto& a, auto& b) { return a.second->seq < b.second->seq; });
    if (oldest->first == video_id) break;
    e->last.erase(oldest);
  }
}

extern "C" mrsp_status mrsp_engine_encode(mrsp_engine* e, const char* video_id,
                                          const float* pixels, int F, int pixels_on_device,
                                          int use_cache, int* hit) {
  return guard([&] {
    MRSP_REQUIRE(e && video_id && pixels, MRSP_INVALID_ARGUMENT, "encode: null argument");
    bool h = false;
    auto entry = e->impl->get_or_encode(video_id, pixels, F, pixels_on_device != 0, use_cache != 0, &h);
    remember(e, video_id, entry);
    if (hit) *hit = h ? 1 : 0;
  });
}

extern "C" mrsp_status mrsp_engine_prefill_logprobs(mrsp_engine* e, const char* video_id,
                                                    const int32_t* question, int n_q,
                                                    const int32_t* resp, const int32_t* lengths,
                                                    int G, int Lmax, int model, float* logprob,
                                                    float* lse, int out_on_device) {
  return guard([&] {
    MRSP_REQUIRE(e && video_id && resp && lengths && logprob && (question || n_q == 0),
                 MRSP_INVALID_ARGUMENT, "prefill: null argument");
    MRSP_REQUIRE(G >= 1, MRSP_INVALID_ARGUMENT, "pad_batch: empty batch");
    auto entry = lookup(e, video_id);
    e->impl->prefill_logprobs(*entry, question, n_q, resp, lengths, G, Lmax, model, logprob, lse,
                              out_on_device != 0);
  });
}

extern "C" mrsp_status mrsp_engine_step(mrsp_engine* e, const char* video_id, const float* pixels,
                                        int F, int pixels_on_device, int use_cache,
                                        const int32_t* question, int n_q, const int32_t* resp,
                                        const int32_t* lengths, int G, int Lmax,
                                        float* logprob_policy, float* logprob_ref, float* kl,
                                        int out_on_device) {
  return guard([&] {
    MRSP_REQUIRE(e && video_id && pixels && resp && lengths && (question || n_q == 0),
                 MRSP_INVALID_ARGUMENT, "step: null argument");
    MRSP_REQUIRE(G >= 1, MRSP_INVALID_ARGUMENT, "pad_batch: empty batch");  // engine.cpp:32
    std::shared_ptr<CacheEntry> entry;
    for (int g = 0; g < G; ++g) {  // one embedding fetch per rollout (grpo.cpp:376-379)
      bool h = false;
      entry = e->impl->get_or_encode(video_id, pixels, F, pixels_on_device != 0, use_cache != 0, &h);
    }
    remember(e, video_id, entry);
    e->impl->group_logprobs(*entry, question, n_q, resp, lengths, G, Lmax, logprob_policy,
                            logprob_ref, kl, out_on_device != 0);
  });
}

extern "C" mrsp_status mrsp_engine_stats(mrsp_engine* e, uint64_t* out6, int reset) {
  return guard([&] {
    Engine& x = *e->impl;
    out6[0] = x.encoder_invocations.load();
    out6[1] = x.cache_hits.load();
    out6[2] = x.cache_misses.load();
    out6[3] = x.gather_bytes.load();
    out6[4] = x.pad_reads.load();
    out6[5] = x.a2a_bytes.load();
    if (reset) {
      x.encoder_invocations = 0;
      x.cache_hits = 0;
      x.cache_misses = 0;
      x.gather_bytes = 0;
      x.pad_reads = 0;
      x.a2a_bytes = 0;
    }
  });
}

extern "C" mrsp_status mrsp_engine_cache(mrsp_engine* e, int op, int arg, uint64_t* size_out) {
  return guard([&] {
    if (op == 1) {
      e->impl->cache_clear();
      std::lock_guard<std::mutex> lock(e->mu);
      e->last.clear();
    } else if (op == 2) {
      e->impl->cache_capacity = arg;
    }
    if (size_out) *size_out = e->impl->cache_size();
  });
}

extern "C" mrsp_status mrsp_engine_generate(mrsp_engine* e, const char* video_id,
                                            const int32_t* question, int n_q, int G, int max_len,
                                            float temperature, uint64_t seed, int32_t* tokens_out,
                                            int32_t* lengths_out, float* old_logprobs_out) {
  return guard([&] {
    MRSP_REQUIRE(e && video_id && (question || n_q == 0) && tokens_out && lengths_out &&
                     old_logprobs_out,
                 MRSP_INVALID_ARGUMENT, "generate: null argument");
    auto entry = lookup(e, video_id);
    e->impl->generate(*entry, question, n_q, G, max_len, temperature, seed, tokens_out,
                      lengths_out, old_logprobs_out);
  });
}

extern "C" mrsp_status mrsp_engine_grpo_backward(mrsp_engine* e, const char* video_id,
                                                 const int32_t* question, int n_q,
                                                 const int32_t* resp, const int32_t* lengths, int G,
                                                 int Lmax, const float* old_logprobs,
                                                 const float* advantages, double clip_eps,
                                                 double kl_beta, int sampled_kl, double* stats4,
                                                 float* logprob_policy) {
  return guard([&] {
    MRSP_REQUIRE(e && video_id && resp && lengths && old_logprobs && advantages && stats4 &&
                     (question || n_q == 0),
                 MRSP_INVALID_ARGUMENT, "grpo_backward: null argument");
    MRSP_REQUIRE(G >= 1, MRSP_INVALID_ARGUMENT, "grpo: empty rollout group");  // grpo.cpp:60
    auto entry = lookup(e, video_id);
    e->impl->grpo_backward(*entry, question, n_q, resp, lengths, G, Lmax, old_logprobs, advantages,
                           clip_eps, kl_beta, sampled_kl, stats4, logprob_policy);
  });
}

extern "C" mrsp_status mrsp_engine_sft_backward(mrsp_engine* e, const char* video_id,
                                                const int32_t* question, int n_q,
                                                const int32_t* resp, const int32_t* lengths, int G,
                                                int Lmax, double* loss_out, float* logprob_policy) {
  return guard([&] {
    MRSP_REQUIRE(e && video_id && resp && lengths && loss_out && (question || n_q == 0),
                 MRSP_INVALID_ARGUMENT, "sft_loss_and_grad: null argument");
    MRSP_REQUIRE(G >= 1, MRSP_INVALID_ARGUMENT, "sft_loss_and_grad: empty targets");
    auto entry = lookup(e, video_id);
    e->impl->sft_backward(*entry, question, n_q, resp, lengths, G, Lmax, loss_out, logprob_policy);
  });
}

extern "C" mrsp_status mrsp_engine_save_grads(mrsp_engine* e, const char* path) {
  return guard([&] {
    MRSP_REQUIRE(e && path, MRSP_INVALID_ARGUMENT, "save_grads: null argument");
    e->impl->save_grads(path);
  });
}

extern "C" mrsp_status mrsp_engine_save_weights(mrsp_engine* e, const char* path) {
  return guard([&] {
    MRSP_REQUIRE(e && path, MRSP_INVALID_ARGUMENT, "save_weights: null argument");
    e->impl->save_weights(path);
  });
}

extern "C" mrsp_status mrsp_engine_load_weights(mrsp_engine* e, const char* path, int part,
                                               const char* prefix) {
  return guard([&] {
    MRSP_REQUIRE(e && path, MRSP_INVALID_ARGUMENT, "load_weights: null argument");
    e->impl->load_weights(path, part, prefix ? prefix : "");
    if (part == 0) {  // embeddings of the old tower are stale
      std::lock_guard<std::mutex> lock(e->mu);
      e->last.clear();
    }
  });
}

extern "C" mrsp_status mrsp_engine_cache_save(mrsp_engine* e, const char* video_id,
                                              const char* path) {
  return guard([&] {
    MRSP_REQUIRE(e && video_id && path, MRSP_INVALID_ARGUMENT, "cache_save: null argument");
    auto entry = lookup(e, video_id);
    e->impl->cache_save(*entry, path);
  });
}

extern "C" mrsp_status mrsp_engine_cache_load(mrsp_engine* e, const char* video_id,
                                              const char* path, int* frames_out) {
  return guard([&] {
    MRSP_REQUIRE(e && video_id && path, MRSP_INVALID_ARGUMENT, "cache_load: null argument");
    auto entry = e->impl->cache_load(video_id, path);
    {
      std::lock_guard<std::mutex> lock(e->mu);
      e->last[video_id] = entry;
    }
    if (frames_out) *frames_out = entry->n_frames;
  });
}

extern "C" mrsp_status mrsp_engine_get_embeddings(mrsp_engine* e, const char* video_id,
                                                  void* host_out, size_t capacity_bytes,
                                                  int* frames_out) {
  return guard([&] {
    MRSP_REQUIRE(e && video_id, MRSP_INVALID_ARGUMENT, "get_embeddings: null argument");
    auto entry = lookup(e, video_id);
    const size_t need = e->impl->embedding_bytes(*entry);
    if (frames_out) *frames_out = entry->n_frames;
    if (!host_out) return;  // size query
    MRSP_REQUIRE(capacity_bytes >= need, MRSP_INVALID_ARGUMENT,
                 "get_embeddings: host buffer holds " + std::to_string(capacity_bytes) +
                     " bytes, the entry needs " + std::to_string(need));
    e->impl->copy_embeddings(*entry, host_out);
  });
}

extern "C" mrsp_status mrsp_engine_profile(mrsp_engine* e, int enable, int cls, double* ms,
                                           int64_t* launches) {
  return guard([&] {
    MRSP_REQUIRE(e, MRSP_INVALID_ARGUMENT, "profile: null engine");
    if (enable >= 0) e->impl->set_profiling(enable != 0);
    if (ms && launches) {
      MRSP_REQUIRE(cls >= 0 && cls <= P_BWD_ATTN, MRSP_INVALID_ARGUMENT, "profile: unknown class");
      long n = 0;
      e->impl->profile_read(cls, ms, &n);
      *launches = n;
    }
  });
}

extern "C" void* mrsp_engine_stream(mrsp_engine* e) { return e ? e->impl->stream() : nullptr; }

extern "C" mrsp_status mrsp_engine_p2p_export(mrsp_engine* e, int max_frames, long max_tokens,
                                              long max_scored, void* blob_out) {
  return mrsp::guard([&] {
    MRSP_REQUIRE(e && e->impl, MRSP_INVALID_ARGUMENT, "null engine");
    std::lock_guard<std::mutex> lock(e->mu);
    e->impl->p2p_export(max_frames, max_tokens, max_scored, blob_out);
  });
}

extern "C" mrsp_status mrsp_engine_p2p_import(mrsp_engine* e, const void* blobs) {
  return mrsp::guard([&] {
    MRSP_REQUIRE(e && e->impl, MRSP_INVALID_ARGUMENT, "null engine");
    std::lock_guard<std::mutex> lock(e->mu);
    e->impl->p2p_import(blobs);
  });
}
