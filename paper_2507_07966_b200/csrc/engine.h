// engine.h — the transformer-shaped MR-SP engine (csrc/engine.cu).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <array>
#include <atomic>
#include <condition_variable>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "comm.h"
#include "mrsp_c.h"
#include "peer.h"

namespace mrsp {

using bf16 = __nv_bfloat16;

// Grow-only device buffer.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) {
    o.p = nullptr;
    o.bytes = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      bytes = o.bytes;
      o.p = nullptr;
      o.bytes = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void release();
  void* ensure(size_t b);
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

struct VisionLayerW {
  float *ln1_w, *ln1_b, *bqkv, *bo, *ln2_w, *ln2_b, *b1, *b2;
  bf16 *wqkv, *wo, *w1, *w2;
};
struct VisionW {
  bf16* patch_w;
  float *patch_b, *pos;
  std::vector<VisionLayerW> layers;
  float *post_w, *post_b, *p1_b, *p2_b;
  bf16 *p1_w, *p2_w;
};
struct LlmLayerW {
  float *attn_norm, *bqkv, *mlp_norm;
  bf16 *wqkv, *wo, *wgu, *wdown;
};
struct LlmW {
  bf16* embed;
  std::vector<LlmLayerW> layers;
  float* final_norm;
  bf16* lm_head;
};

struct HeadSplit {
  int q_lo, q_hi, kv_lo, kv_hi, q_per_kv;
  // Query-row split (SP > n_kv, peer-memory transport): the rparts ranks
  // sharing a kv head each take ALL its query heads over part rpart of the
  // 256-row query blocks (attn_row_part), instead of splitting the heads 4+3.
  int rparts = 1, rpart = 0;
  int nq() const { return q_hi - q_lo; }
  int nkv() const { return kv_hi - kv_lo; }
};

HeadSplit head_split(int nq, int nkv, int k, int r, bool row_split = false);

// fp32 elements per chunk of the cross-process weight-gradient sum (peer mesh
// staging: one slot per rank, 16 MB each)
constexpr long kGradReduceChunk = 4L << 20;

// Column stride of one vision head in the engine's QKV / attention-output
// storage: the real head dim (SigLIP 72: unpadded GEMMs; the attention's 3-D
// TMA boxes zero-fill 72 -> 128 on chip) when its rows are 16-byte multiples,
// else 128 (zero-padded in HBM). MRSP_VISION_PAD=1 forces 128 (read when an
// engine is created).
int vision_head_stride(const mrsp_model_config& c);

// One SP rank living in this process (k of them in loopback mode, 1 with NCCL).
struct RankCtx {
  int g = 0;  // global SP rank
  HeadSplit hs{};
  // stage 1
  DevBuf pix, patches, vh, vxn, vqkv, vo, vmid, pout;
  // stage 2
  DevBuf h, xn, qkv, qh, oh, ol, act, pos, pad, scored_idx, xs, xs2, lp, ws, send, recv;
  long b = 0, e = 0;  // token range
  int n_scored = 0;
  // spread LM head: this rank computes the scored tokens [lm_lo, lm_lo + lm_n)
  // of the group (plan_shards over the scored tokens), its own scored tokens
  // being [sc_lo, sc_lo + n_scored); lm_idx = [targets | slots] of its slice,
  // lmx = [2][lm_n][d] landing rows (virtual ranks)
  long sc_lo = 0, lm_lo = 0;
  int lm_n = 0;
  DevBuf lm_idx, lmx;
};

struct CacheEntry {
  std::mutex m;
  std::condition_variable cv;
  bool ready = false;
  bool failed = false;
  std::string error;
  std::shared_ptr<DevBuf> emb;  // [F*T][dim] bf16, all frames (gathered)
  int n_frames = 0;
  uint64_t seq = 0;
};

class Engine {
 public:
  Engine(const mrsp_model_config& cfg, int sp_degree, int proc_rank, int n_procs,
         uint64_t vision_seed, uint64_t policy_seed, uint64_t ref_seed, int with_ref,
         const void* nccl_id);
  ~Engine();

  // Stage 1 with the exactly-once cache (engine.cpp:155-197 protocol).
  std::shared_ptr<CacheEntry> get_or_encode(const std::string& id, const float* pixels, int F,
                                            bool on_device, bool use_cache, bool* hit);
  // Stage 2 for one model over the packed GRPO group; lp_out has sum(lengths)
  // entries (host or device per lp_on_device).
  void prefill_logprobs(const CacheEntry& emb, const int32_t* question, int n_q,
                        const int32_t* resp, const int32_t* lengths, int G, int Lmax, int model,
                        float* lp_out, float* lse_out, bool out_on_device);
  // Policy + reference passes and the fused dual LM head (log-probs of both
  // models and the exact per-token KL in one vocabulary sweep).
  void group_logprobs(const CacheEntry& emb, const int32_t* question, int n_q,
                      const int32_t* resp, const int32_t* lengths, int G, int Lmax,
                      float* lp_policy, float* lp_ref, float* kl, bool out_on_device);

  const mrsp_model_config& cfg() const { return cfg_; }
  int tokens_per_frame() const { return (cfg_.image_size / cfg_.patch) * (cfg_.image_size / cfg_.patch); }
  int sp() const { return k_; }
  cudaStream_t stream() const { return stream_; }
  std::vector<RankCtx>& ranks() { return ranks_; }

  // counters (EngineStats, engine.hpp:27-41, plus device traffic)
  std::atomic<uint64_t> encoder_invocations{0}, cache_hits{0}, cache_misses{0}, gather_bytes{0},
      pad_reads{0}, a2a_bytes{0};
  size_t cache_size();
  void cache_clear();
  // Rollout generation (policy.cpp:121-157): G rows sampled
  // autoregressively from the policy after the prompt [video | question],
  // reusing the cached video embeddings and the prompt's K/V (one prefix
  // prefill, then decode steps). SP = 1, one process.
  void generate(const CacheEntry& emb, const int32_t* question, int n_q, int G, int max_len,
                float temperature, uint64_t seed, int32_t* tokens_out, int32_t* lengths_out,
                float* old_lp_out);
  // weights to / from safetensors with HF names (csrc/weights_io.cpp); part 0 =
  // vision tower + projector, 1 = policy LLM, 2 = reference LLM
  void save_weights(const std::string& path);
  void load_weights(const std::string& path, int part, const std::string& prefix);
  // cache persistence: a gathered video's embeddings to / from a file
  void cache_save(const CacheEntry& e, const std::string& path);
  std::shared_ptr<CacheEntry> cache_load(const std::string& id, const std::string& path);
  int cache_capacity = 0;  // 0 = unbounded

  // GRPO gradient of the policy LLM (grpo_gradient,
  // grpo.cpp:122-206, through the transformer-shaped decoder): both prefill
  // passes (the policy's with its layer inputs kept), the fused dual LM head,
  // then the backward of the LM head, the final norm, every decoder layer
  // (recomputed from its kept input) and the text embeddings. The vision tower
  // and projector are frozen (the reference differentiates only the policy).
  // Host in: old_lp [sum(lengths)], adv [G]; host out: stats4 = {objective,
  // mean_kl, clip_fraction, tokens}, optional lp [sum(lengths)]. Gradients
  // stay on the device (grads_) until save_grads.
  void grpo_backward(const CacheEntry& emb, const int32_t* question, int n_q,
                     const int32_t* resp, const int32_t* lengths, int G, int Lmax,
                     const float* old_lp, const float* adv, double clip_eps, double kl_beta,
                     int sampled_kl, double* stats4, float* lp_out);
  // SFT loss and gradient (sft_loss_and_grad, grpo.cpp:208-223) of the policy
  // over G teacher-forced rows: loss = mean over all row tokens of -log pi(y)
  void sft_backward(const CacheEntry& emb, const int32_t* question, int n_q,
                    const int32_t* resp, const int32_t* lengths, int G, int Lmax,
                    double* loss_out, float* lp_out);
  // the last grpo_backward's gradients as an F32 safetensors file (policy
  // tensor names, csrc/weights_io.cpp)
  void save_grads(const std::string& path);

  // profiling: CUDA-event time per kernel class
  void set_profiling(bool on);
  void profile_read(int cls, double* ms, long* launches);
  size_t embedding_bytes(const CacheEntry& e) const;
  void copy_embeddings(const CacheEntry& e, void* host_out);

 private:
  friend struct Prof;
  void init_weights(uint64_t vision_seed, uint64_t policy_seed, uint64_t ref_seed, int with_ref);
  void encode_rank(RankCtx& R, const float* pixels, bool on_device, int F, long fb, long fe,
                   bf16* out);
  void a2a_forward(int L);
  void a2a_backward(int L);
  void prepare_group(const CacheEntry& emb, const int32_t* question, int n_q,
                     const int32_t* resp, const int32_t* lengths, int G, int Lmax);
  void run_pass(const CacheEntry& emb, int model, int xs_slot);
  void backward_pass(int mode, const CacheEntry& emb, const int32_t* question, int n_q,
                     const int32_t* resp, const int32_t* lengths, int G, int Lmax,
                     const float* old_lp, const float* adv, double clip_eps, double kl_beta,
                     int sampled_kl, double* stats4, float* lp_out);
  // backward: per-layer input hidden states kept by run_pass (per local rank,
  // [layers][n][d] fp32; empty = off), the per-rank backward workspaces and
  // the fp32 gradients in the engine's weight layout
  std::vector<float*> stash_;
  std::vector<DevBuf> stash_bufs_, bwd_ws_;
  // ... and, when they fit (bwd_stash_attention), each layer's attention
  // output O ([layers][n][nq 128] bf16, sequence shard) and log-sum-exp
  // ([layers][nq_r][stash_lse_ld_] fp32, head shard), so the backward skips
  // the attention recompute
  std::vector<bf16*> stash_o_;
  std::vector<float*> stash_lse_;
  std::vector<DevBuf> stash_attn_bufs_;
  int stash_lse_ld_ = 0;
  DevBuf grad_buf_, bwd_group_ws_;
  LlmW grads_{};  // fp32 storage typed as the weight struct (see save_grads)
  bool have_grads_ = false;
  // prefix K/V capture for generation (run_pass copies rows [0, Lp) of every
  // layer's post-RoPE K and V when set): [layers][Lp][2 n_kv 128] bf16
  DevBuf kv_prefix_;
  bool capture_kv_ = false;
  void finish_group(int nvec, float* const* outs, bool out_on_device);

  struct GroupState {
    int n_q = 0, G = 0, Lmax = 0;
    long n_frame_tok = 0, Lp = 0, Ltot = 0, total_scored = 0, stride = 0;
    const int32_t *d_question = nullptr, *d_resp = nullptr, *d_len = nullptr;
    float* full = nullptr;  // group-ordered output vectors (stride floats each)
  } grp_;

  mrsp_model_config cfg_;
  int k_, proc_rank_, n_procs_, device_ = 0;
  cudaStream_t stream_ = nullptr;
  std::unique_ptr<Nccl> nccl_;
  std::vector<RankCtx> ranks_;
  DevBuf wbuf_;  // all weights
  VisionW vis_{};
  LlmW llm_[2]{};
  bool has_ref_ = false;
  int vhd_pad_ = 128;
  std::vector<long> token_b_, token_e_;  // current stage-2 plan
  // fused Ulysses routing (GEMM_EPI_QKV_SCATTER / attention O scatter): device
  // [inv_freq 64 f32 | route int2[2 * n_blocks] | peer_ld int[8] | peer_base ptr[8]]
  DevBuf route_buf_;
  float* d_inv_freq_ = nullptr;
  int2* d_route_ = nullptr;
  int* d_peer_ld_ = nullptr;
  void** d_peer_base_ = nullptr;
  std::array<void*, 8> h_peer_base_{};
  void build_routes(const float* inv_freq);
  bool fused_a2a() const { return !nccl_; }
  // query-row split of a shared kv head's query heads (HeadSplit::rparts):
  // the fused transports at SP > n_kv, unless MRSP_ULYSSES_SPLIT=heads
  bool row_split_ = false;
  int vstride_ = 128;  // vision_head_stride(cfg_), fixed at construction
  HeadSplit split_of(int p) const {
    return head_split(cfg_.n_q_heads, cfg_.n_kv_heads, k_, p, row_split_);
  }
  // bytes this group's fused all-to-alls move off each local rank per layer
  std::vector<uint64_t> a2a_fwd_bytes_, a2a_bwd_bytes_;
  std::vector<int2> route_h_;  // host copy of d_route_
  // LM head over plan_shards of the scored tokens instead of on the shards
  // that own them (the response rows are the sequence tail, i.e. the last
  // shard): the final-norm rows move to their computing rank first
  bool spread_lm() const { return k_ > 1 && fused_a2a(); }
  // rows X of local rank R's LM-head slice for model slot m (0: xs, 1: xs2)
  const void* lm_rows(RankCtx& R, int m);
  void lm_exchange(int n_models);
  void plan_a2a_bytes();
  // one process per GPU over CUDA-IPC peer memory (no NCCL id given)
  std::unique_ptr<PeerMesh> mesh_;
  // head-shard / sequence-shard output buffers of SP rank p (a virtual rank's
  // own buffer, or a peer's mapped landing buffer)
  void* qh_dst(int p) { return mesh_ ? mesh_->qh(p) : ranks_[p].qh.p; }
  void* ol_dst(int p) { return mesh_ ? mesh_->ol(p) : ranks_[p].ol.p; }

 public:
  size_t p2p_export(int max_frames, long max_tokens, long max_scored, void* blob);
  void p2p_import(const void* blobs);

 private:
  std::mutex cache_mu_;
  std::map<std::string, std::shared_ptr<CacheEntry>> cache_;
  std::vector<std::shared_ptr<DevBuf>> entry_pool_;  // recycled entry buffers (run_mu_)
  std::shared_ptr<DevBuf> entry_buffer(size_t bytes);
  uint64_t cache_seq_ = 0;
  std::mutex run_mu_;  // one stage at a time per engine
  // profiling
  bool prof_ = false;
  struct Ev {
    int cls;
    cudaEvent_t a, b;
  };
  std::vector<Ev> ev_pending_;
  std::vector<cudaEvent_t> ev_pool_;
  static constexpr int kProfClasses = 9;
  double prof_ms_[kProfClasses] = {0};
  long prof_n_[kProfClasses] = {0};
  void prof_begin(int cls, cudaEvent_t* a);
  void prof_end(int cls, cudaEvent_t a);
  void prof_collect();

 public:
  DevBuf io_;  // step I/O staging
};

std::array<std::array<int, 3>, 3> ulysses_blocks(int nq, int nkv, const HeadSplit& hs);

// CUDA-event time of one kernel class while profiling is on (scoped).
struct Prof {
  Engine& e;
  int cls;
  cudaEvent_t a = nullptr;
  Prof(Engine& en, int c) : e(en), cls(c) { e.prof_begin(cls, &a); }
  ~Prof() {
    if (a) e.prof_end(cls, a);
  }
};

enum { P_ATTN = 0, P_GEMM = 1, P_VISION = 2, P_LMHEAD = 3, P_COMM = 4, P_MISC = 5,
       P_DECODE_GRAPH = 6, P_BACKWARD = 7, P_BWD_ATTN = 8 };

}  // namespace mrsp
