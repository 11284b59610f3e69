// engine_bwd.cu — the GRPO gradient through the transformer-shaped SP prefill
// (SURVEY §8f rank 3). The reference computes it analytically for its toy
// policy: grpo_gradient (grpo.cpp:122-206) builds g = dJ/dlogits per scored
// position — the clipped-ratio term and the exact-KL (or k3) term — and
// GradAccumulator::add_position (policy.cpp:195-260) back-propagates it into
// the policy parameters. Here the same g drives the backward of the Qwen-shaped
// decoder stack:
//
//   LM head      G = dJ/dlogits recomputed per 128 x 256 vocabulary tile from both
//                models' final hidden rows (lmhead_dual_dlogits), then
//                dX = G W (dgrad) and dW_lm = G^T X (wgrad) on the tcgen05 GEMM
//                with MN-major operands
//   final norm   RMSNorm backward at the scored positions
//   layer l      recomputed from its kept input h_l (activation checkpointing:
//                the forward keeps one fp32 [n][d] per layer): RMSNorm, QKV +
//                RoPE, attention (with its log-sum-exp — or, when they fit,
//                the O and log-sum-exp the policy pass kept), O projection, RMSNorm;
//                then  d act = dh W_down;  the gate/up GEMM again with the
//                SwiGLU-backward epilogue (dgate | dup, and act);  wgrads of
//                W_down, W_gate|up;  dx = dgu W_gu;  RMSNorm backward;  dO =
//                dh W_o;  wgrad W_o;  attention backward (dQ, dK, dV);  RoPE
//                backward (rotation by -pos);  bias grad;  wgrad / dgrad of
//                W_qkv;  RMSNorm backward
//   embeddings   dE[token] = sum of dh over the token's text positions
//
// The vision tower and projector are frozen (the reference differentiates only
// the policy parameters, policy.hpp:39-53). Every reduction runs in a fixed
// order, so the gradients are deterministic.
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <map>
#include <vector>

#include "attention.h"
#include "backward.h"
#include "common.h"
#include "engine.h"
#include "gemm.h"
#include "misc.h"

namespace mrsp {

namespace {
struct Carve {
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

void Engine::grpo_backward(const CacheEntry& emb, const int32_t* question, int n_q,
                           const int32_t* resp, const int32_t* lengths, int G, int Lmax,
                           const float* old_lp, const float* adv, double clip_eps, double kl_beta,
                           int sampled_kl, double* stats4, float* lp_out) {
  MRSP_REQUIRE(old_lp && adv && stats4 && lengths, MRSP_INVALID_ARGUMENT,
               "grpo_backward: null argument");
  MRSP_REQUIRE(clip_eps >= 0.0, MRSP_INVALID_ARGUMENT, "grpo_backward: clip_eps < 0");
  // check_group (grpo.cpp:57-66): every rollout has tokens
  MRSP_REQUIRE(G >= 1 && G <= 1024, MRSP_INVALID_ARGUMENT, "grpo: empty rollout group");
  for (int r = 0; r < G; ++r)
    MRSP_REQUIRE(lengths[r] >= 1, MRSP_INVALID_ARGUMENT, "grpo: empty rollout");
  MRSP_REQUIRE(has_ref_ || kl_beta == 0.0, MRSP_INVALID_ARGUMENT,
               "grpo_backward: the KL term needs a separate reference model");
  backward_pass(0, emb, question, n_q, resp, lengths, G, Lmax, old_lp, adv, clip_eps, kl_beta,
                sampled_kl, stats4, lp_out);
}

void Engine::sft_backward(const CacheEntry& emb, const int32_t* question, int n_q,
                          const int32_t* resp, const int32_t* lengths, int G, int Lmax,
                          double* loss_out, float* lp_out) {
  MRSP_REQUIRE(loss_out, MRSP_INVALID_ARGUMENT, "sft_loss_and_grad: null argument");
  double st[4] = {0, 0, 0, 0};
  backward_pass(1, emb, question, n_q, resp, lengths, G, Lmax, nullptr, nullptr, 0.0, 0.0, 0, st,
                lp_out);
  *loss_out = st[0];
}

// mode 0: GRPO objective (gradient of J, ascent direction, as grpo_gradient);
// mode 1: SFT loss = mean over the rows' tokens of -log pi(y) (gradient of the
// loss, as sft_loss_and_grad, grpo.cpp:208-223; the reference pass is skipped).
void Engine::backward_pass(int mode, const CacheEntry& emb, const int32_t* question, int n_q,
                           const int32_t* resp, const int32_t* lengths, int G, int Lmax,
                           const float* old_lp, const float* adv, double clip_eps, double kl_beta,
                           int sampled_kl, double* stats4, float* lp_out) {
  const auto& c = cfg_;
  const int d = c.dim, nq = c.n_q_heads, nkv = c.n_kv_heads, mlp = c.mlp, V = c.vocab;
  const int Cqkv = (nq + 2 * nkv) * 128, Cq = nq * 128, NL = c.layers;
  MRSP_REQUIRE(!nccl_, MRSP_INVALID_ARGUMENT,
               "grpo_backward: built on the peer-memory transport (one process with virtual SP "
               "ranks, or one process per GPU over CUDA IPC), not on NCCL");
  MRSP_REQUIRE(!mesh_ || mesh_->ready(), MRSP_INVALID_ARGUMENT,
               "grpo_backward: p2p export / import first");
  MRSP_REQUIRE(d % 8 == 0 && mlp % 128 == 0 && V % 8 == 0, MRSP_INVALID_ARGUMENT,
               "grpo_backward: unsupported model geometry");
  std::lock_guard<std::mutex> run(run_mu_);
  cudaStream_t s = stream_;
  prepare_group(emb, question, n_q, resp, lengths, G, Lmax);
  const GroupState& g = grp_;
  const long Ltot = g.Ltot;
  const int S = static_cast<int>(g.total_scored);
  MRSP_REQUIRE(S >= 1, MRSP_INVALID_ARGUMENT, "grpo_backward: the group has no scored token");
  const int K = k_;                                      // SP degree
  const int m_kv = K > nkv ? K / nkv : 1;                // ranks sharing one kv head
  const int NLOC = static_cast<int>(ranks_.size());      // SP ranks in this process
  if (mesh_)
    MRSP_REQUIRE(Ltot <= mesh_->caps().tokens && S <= mesh_->caps().scored, MRSP_INVALID_ARGUMENT,
                 "p2p: group exceeds the exported capacities");
  // every global rank's scored tokens [sc_lo, sc_lo + n_sc) in group order
  // (scored tokens are position-ordered): where the LM-head slices' dX rows go
  std::vector<long> sc_lo(K, 0), n_sc(K, 0);
  for (int r = 0; r < G; ++r)
    for (int j = 0; j < lengths[r]; ++j) {
      const long pos = g.Lp + static_cast<long>(r) * Lmax + j;
      int p = 0;
      while (p + 1 < K && pos >= token_b_[p + 1]) ++p;
      ++n_sc[p];
    }
  for (int p = 1; p < K; ++p) sc_lo[p] = sc_lo[p - 1] + n_sc[p - 1];

  // ---- gradient storage: fp32 in the engine's weight layout, zeroed per call
  // (every SP rank adds its tokens' share, in rank order: deterministic) -----
  size_t grad_bytes = 0;
  {
    auto add = [&](size_t elems) { grad_bytes += (elems * 4 + 255) & ~size_t(255); };
    add(static_cast<size_t>(V) * d);
    for (int l = 0; l < NL; ++l) {
      add(d); add(static_cast<size_t>(Cqkv) * d); add(Cqkv); add(static_cast<size_t>(d) * Cq);
      add(d); add(static_cast<size_t>(2) * mlp * d); add(static_cast<size_t>(d) * mlp);
    }
    add(d);
    add(static_cast<size_t>(V) * d);
  }
  if (!grad_buf_.p) {
    grad_buf_.ensure(grad_bytes);
    Carve cv{static_cast<uint8_t*>(grad_buf_.p)};
    grads_.embed = reinterpret_cast<bf16*>(cv.take<float>(static_cast<size_t>(V) * d));
    grads_.layers.resize(NL);
    for (int l = 0; l < NL; ++l) {
      auto& L = grads_.layers[l];
      L.attn_norm = cv.take<float>(d);
      L.wqkv = reinterpret_cast<bf16*>(cv.take<float>(static_cast<size_t>(Cqkv) * d));
      L.bqkv = cv.take<float>(Cqkv);
      L.wo = reinterpret_cast<bf16*>(cv.take<float>(static_cast<size_t>(d) * Cq));
      L.mlp_norm = cv.take<float>(d);
      L.wgu = reinterpret_cast<bf16*>(cv.take<float>(static_cast<size_t>(2) * mlp * d));
      L.wdown = reinterpret_cast<bf16*>(cv.take<float>(static_cast<size_t>(d) * mlp));
    }
    grads_.final_norm = cv.take<float>(d);
    grads_.lm_head = reinterpret_cast<bf16*>(cv.take<float>(static_cast<size_t>(V) * d));
  }
  have_grads_ = false;
  MRSP_CUDA(cudaMemsetAsync(grad_buf_.p, 0, grad_bytes, s));

  // ---- group-wide vectors (group order) -------------------------------------
  float *lp_f, *lpr_f, *kl_f, *coef_f, *old_f, *adv_f;
  double* d_stats;
  {
    auto layout = [&](Carve& cv) {
      lp_f = cv.take<float>(S);
      lpr_f = cv.take<float>(S);
      kl_f = cv.take<float>(S);
      coef_f = cv.take<float>(S);
      old_f = cv.take<float>(S);
      adv_f = cv.take<float>(G);
      d_stats = cv.take<double>(4);
    };
    Carve sizing{nullptr};
    layout(sizing);
    bwd_group_ws_.ensure(sizing.off);
    Carve cv{static_cast<uint8_t*>(bwd_group_ws_.p)};
    layout(cv);
  }

  // ---- per-rank workspaces --------------------------------------------------
  struct RW {
    float *hm, *dh, *dx, *dxs_own, *lp, *lpr, *kl, *lsep, *lser, *stat_lse, *stat_D, *dxs;
    bf16 *dhb, *xn1, *dact, *dgu, *dO, *dqkv, *Gl, *doh, *dqkvh;
    float *slots, *dkv32;  // shared kv heads: fp32 dk | dv partials
    float* dseq;  // [nq][ld_dseq] row dots of dO and O on the sequence side
    int ld_dseq;
    int* negpos;
    void *ws, *dws;
    int ld_stat;
  };
  std::vector<RW> rw(NLOC);
  stash_bufs_.resize(NLOC);
  bwd_ws_.resize(NLOC);
  for (int r = 0; r < NLOC; ++r) {
    RankCtx& R = ranks_[r];
    const int n = static_cast<int>(R.e - R.b);
    const size_t nd = static_cast<size_t>(n) * d;
    const int nqr = R.hs.nq(), Cr = (R.hs.nq() + 2 * R.hs.nkv()) * 128;
    const int lm = std::max(R.lm_n, 1), own = std::max(R.n_scored, 1);
    const long Lh = K == 1 ? n : Ltot;  // rows of the attention (head-shard) problem
    const int ld_stat = static_cast<int>((Lh + 3) / 4 * 4);
    const size_t ws_norm = rmsnorm_bwd_workspace_bytes(std::max(n, own), d);
    const size_t ws_col = colsum_workspace_bytes(n, Cqkv);
    const size_t dual_ws = lmhead_dual_workspace_bytes(lm, V);
    RW& w = rw[r];
    // one layout function, run once to size the buffer and once to carve it
    auto layout = [&](Carve& cv) {
      w.hm = cv.take<float>(nd);
      w.dh = cv.take<float>(nd);
      w.dx = cv.take<float>(nd);
      w.dhb = cv.take<bf16>(nd);
      w.xn1 = cv.take<bf16>(nd);
      w.dact = cv.take<bf16>(static_cast<size_t>(n) * mlp);
      w.dgu = cv.take<bf16>(static_cast<size_t>(n) * 2 * mlp);
      w.dO = cv.take<bf16>(static_cast<size_t>(n) * Cq);
      // dq | dk | dv of the shard: a peer-mesh landing buffer across processes
      w.dqkv = mesh_ ? static_cast<bf16*>(mesh_->dqkv(R.g)) : cv.take<bf16>(static_cast<size_t>(n) * Cqkv);
      w.stat_lse = cv.take<float>(static_cast<size_t>(std::max(nqr, 1)) * ld_stat);
      w.stat_D = cv.take<float>(static_cast<size_t>(std::max(nqr, 1)) * ld_stat);
      w.negpos = cv.take<int>(n);
      w.Gl = cv.take<bf16>(static_cast<size_t>(lm) * V);
      w.dxs = cv.take<float>(static_cast<size_t>(lm) * d);
      w.dxs_own = mesh_ ? mesh_->dxs(R.g) : cv.take<float>(static_cast<size_t>(own) * d);
      w.lp = cv.take<float>(lm);
      w.lpr = cv.take<float>(lm);
      w.kl = cv.take<float>(lm);
      w.lsep = cv.take<float>(lm);
      w.lser = cv.take<float>(lm);
      w.ws = cv.take<uint8_t>(std::max(ws_norm, ws_col));
      w.dws = cv.take<uint8_t>(dual_ws);
      w.doh = mesh_ ? static_cast<bf16*>(mesh_->doh(R.g))
            : K > 1 ? cv.take<bf16>(static_cast<size_t>(Ltot) * std::max(nqr, 1) * 128) : nullptr;
      w.dqkvh = K > 1 ? cv.take<bf16>(static_cast<size_t>(Ltot) * Cr) : nullptr;
      w.ld_dseq = (n + 3) / 4 * 4;
      w.dseq = K > 1 ? cv.take<float>(static_cast<size_t>(nq) * w.ld_dseq) : nullptr;
      // dk | dv partials of kv heads shared by m ranks, one slot per sharer
      w.slots = (K > 1 && m_kv > 1)
                    ? (mesh_ ? static_cast<float*>(mesh_->kv_slots(R.g))
                             : cv.take<float>(static_cast<size_t>(m_kv) * n * 2 * nkv * 128))
                    : nullptr;
      w.dkv32 = (K > 1 && m_kv > 1)
                    ? cv.take<float>(static_cast<size_t>(Ltot) * 2 * std::max(R.hs.nkv(), 1) * 128)
                    : nullptr;
      if (mesh_) w.stat_D = mesh_->dh_stat(R.g);  // routed by every sequence rank
    };
    Carve sizing{nullptr};
    layout(sizing);
    bwd_ws_[r].ensure(sizing.off);
    Carve cv{static_cast<uint8_t*>(bwd_ws_[r].p)};
    layout(cv);
    w.ld_stat = ld_stat;
    stash_bufs_[r].ensure(std::max<size_t>(static_cast<size_t>(NL) * nd * 4, 256));
  }
  // The policy pass also keeps every layer's attention output O and its
  // log-sum-exp when they fit, so the layer recompute below skips the
  // attention (MRSP_BWD_STASH_ATTN=0 / 1: never / always; default: when the
  // largest rank's share is at most a quarter of the device). The decision
  // uses only global sizes and the device's total memory, so every process of
  // a mesh of identical GPUs takes the same one (the peer mesh is one node's
  // GPUs; a rank deciding differently would not send its O rows).
  const int ld_keep = static_cast<int>((Ltot + 3) / 4 * 4);
  bool keep_attn = false;
  std::vector<size_t> o_keep_bytes(NLOC, 0);
  {
    const char* env = std::getenv("MRSP_BWD_STASH_ATTN");
    long n_max = 0;
    int nq_max = 1;
    for (int p = 0; p < K; ++p) {
      n_max = std::max(n_max, token_e_[p] - token_b_[p]);
      nq_max = std::max(nq_max, split_of(p).nq());
    }
    const size_t per_rank = static_cast<size_t>(NL) * n_max * Cq * 2 +
                            static_cast<size_t>(NL) * nq_max * ld_keep * 4;
    size_t free_b = 0, total_b = 0;
    MRSP_CUDA(cudaMemGetInfo(&free_b, &total_b));
    keep_attn = env && std::string(env) == "1"
                    ? true
                    : !(env && std::string(env) == "0") && per_rank * NLOC <= total_b / 4;
  }
  stash_attn_bufs_.resize(NLOC);
  if (keep_attn)
    for (int r = 0; r < NLOC; ++r) {
      const size_t n = static_cast<size_t>(ranks_[r].e - ranks_[r].b);
      o_keep_bytes[r] = (static_cast<size_t>(NL) * n * Cq * 2 + 255) / 256 * 256;
      stash_attn_bufs_[r].ensure(o_keep_bytes[r] + static_cast<size_t>(NL) *
                                                       std::max(ranks_[r].hs.nq(), 1) * ld_keep * 4);
    }
  auto o_kept = [&](int r, int l) {
    return static_cast<bf16*>(stash_attn_bufs_[r].p) +
           static_cast<size_t>(l) * (ranks_[r].e - ranks_[r].b) * Cq;
  };
  auto lse_kept = [&](int r, int l) {
    return reinterpret_cast<float*>(static_cast<uint8_t*>(stash_attn_bufs_[r].p) + o_keep_bytes[r]) +
           static_cast<size_t>(l) * std::max(ranks_[r].hs.nq(), 1) * ld_keep;
  };

  // Ulysses routing of the backward (every global rank's buffers; across
  // processes the peers' landing buffers)
  RouteArgs ra{};
  if (K > 1) {
    MRSP_REQUIRE(K <= 8, MRSP_INVALID_ARGUMENT, "grpo_backward: at most 8 SP ranks");
    ra.K = K;
    ra.nq = nq;
    ra.nkv = nkv;
    ra.L = Ltot;
    ra.n_blocks = static_cast<int>((Ltot + ATTN_ROW_BLOCK - 1) / ATTN_ROW_BLOCK);
    for (int p = 0; p < K; ++p) {
      const HeadSplit hp = split_of(p);
      RouteRank& q = ra.r[p];
      q.q_lo = hp.q_lo;
      q.q_hi = hp.q_hi;
      q.kv_lo = hp.kv_lo;
      q.kv_hi = hp.kv_hi;
      q.rparts = hp.rparts;
      q.rpart = hp.rpart;
      q.slot = m_kv > 1 ? p % m_kv : 0;
      q.b = token_b_[p];
      q.e = token_e_[p];
      q.ld_stat = static_cast<int>((Ltot + 3) / 4 * 4);
      if (mesh_) {
        q.doh = mesh_->doh(p);
        q.Dh = mesh_->dh_stat(p);
        q.dqkv = mesh_->dqkv(p);
        q.slots = mesh_->kv_slots(p);
      } else {
        q.doh = rw[p].doh;
        q.Dh = rw[p].stat_D;
        q.dqkv = rw[p].dqkv;
        q.slots = rw[p].slots;
      }
    }
    // a kv head shared by m ranks must be shared as a query-row split or as a
    // split of its query heads; either way each sharer owns one slot
    for (int p = 0; p < K; ++p)
      MRSP_REQUIRE(m_kv == 1 || (ra.r[p].kv_hi - ra.r[p].kv_lo == 1 && ra.r[p].kv_lo == p / m_kv &&
                                 (ra.r[p].rparts == m_kv || ra.r[p].rparts == 1)),
                   MRSP_INVALID_ARGUMENT, "grpo_backward: unsupported head split");
  }

  // ---- forward: reference pass, then the policy pass keeping layer inputs --
  if (mode == 0) run_pass(emb, 1, 1);  // xs2 = reference final-norm rows
  stash_.resize(NLOC);
  for (int r = 0; r < NLOC; ++r) stash_[r] = stash_bufs_[r].as<float>();
  if (keep_attn) {
    stash_o_.resize(NLOC);
    stash_lse_.resize(NLOC);
    for (int r = 0; r < NLOC; ++r) {
      stash_o_[r] = o_kept(r, 0);
      stash_lse_[r] = lse_kept(r, 0);
    }
    stash_lse_ld_ = ld_keep;
  }
  auto unstash = [&] {
    stash_.clear();
    stash_o_.clear();
    stash_lse_.clear();
    stash_lse_ld_ = 0;
  };
  try {
    run_pass(emb, 0, 0);  // xs = policy final-norm rows; h = h_L of every shard
  } catch (...) {
    unstash();
    throw;
  }
  unstash();
  lm_exchange(mode == 0 ? 2 : 1);  // the final-norm rows to the LM-head slices (spread LM head)
  const LlmW& W = llm_[0];
  // SFT has no reference model: the dual head runs the policy against itself
  // (KL 0, the same log-partition twice)
  const LlmW& Wr = llm_[mode == 0 ? 1 : 0];
  const int ref_slot = mode == 0 ? 1 : 0;
  {
    Prof pl(*this, P_LMHEAD);
    if (mesh_) {  // the group vectors live in every rank's landing buffer
      const long stride = mesh_->caps().scored + 16;
      lp_f = mesh_->lp(ranks_[0].g);
      lpr_f = lp_f + stride;
      kl_f = lp_f + 2 * stride;
      mesh_->barrier(s);  // every rank has read the previous group's outputs
    }
    for (int r = 0; r < NLOC; ++r) {
      RankCtx& R = ranks_[r];
      if (R.lm_n == 0) continue;
      RW& w = rw[r];
      const size_t dual_ws = lmhead_dual_workspace_bytes(R.lm_n, V);
      lmhead_dual_logprob_kl_lse(lm_rows(R, 0), W.lm_head, lm_rows(R, ref_slot), Wr.lm_head, R.lm_n, V, d,
                                 R.lm_idx.as<int32_t>(), w.lp, w.lpr, w.kl, w.lsep, w.lser, w.dws,
                                 dual_ws, s);
      // slices are contiguous in group order; across processes, into every rank's copy
      const size_t off = static_cast<size_t>(R.lm_lo), bytes = static_cast<size_t>(R.lm_n) * 4;
      for (int p = 0; p < (mesh_ ? K : 1); ++p) {
        float* base = mesh_ ? mesh_->lp(p) : lp_f;
        const long stride = mesh_ ? mesh_->caps().scored + 16 : 0;
        float* dst[3] = {base, mesh_ ? base + stride : lpr_f, mesh_ ? base + 2 * stride : kl_f};
        const float* src[3] = {w.lp, w.lpr, w.kl};
        for (int v = 0; v < 3; ++v)
          MRSP_CUDA(cudaMemcpyAsync(dst[v] + off, src[v], bytes, cudaMemcpyDeviceToDevice, s));
      }
    }
    if (mesh_) mesh_->barrier(s);  // every slice has landed
  }
  if (mode == 0) {
    MRSP_CUDA(cudaMemcpyAsync(old_f, old_lp, static_cast<size_t>(S) * 4, cudaMemcpyHostToDevice, s));
    MRSP_CUDA(cudaMemcpyAsync(adv_f, adv, static_cast<size_t>(G) * 4, cudaMemcpyHostToDevice, s));
    grpo_stats(lp_f, old_f, lpr_f, kl_f, adv_f, g.d_len, G, clip_eps, kl_beta, sampled_kl, d_stats, s);
  }
  {
  Prof pb(*this, P_BACKWARD);
  if (mode == 0)
    grpo_token_coeffs(lp_f, old_f, lpr_f, adv_f, g.d_len, G, S, clip_eps, kl_beta, sampled_kl,
                      coef_f, s);
  else  // d(-mean log pi(y))/dlogits = (pi - onehot(y)) / n  (grpo.cpp:217-219)
    fill_f32(coef_f, S, -1.0f / static_cast<float>(S), s);
  const float kw = (mode != 0 || sampled_kl || kl_beta == 0.0) ? 0.f : static_cast<float>(-kl_beta / S);
  auto gemm_mn = [&](const void* A, int lda, int a_mn, const void* B, int ldb, int b_mn, void* C,
                     int ldc, int M, int N, int Kd, int epi) {
    if (M <= 0 || N <= 0 || Kd <= 0) return;
    GemmArgs ga{A, B, C, M, N, Kd, lda, ldb, ldc, epi, nullptr, nullptr, 0};
    if (epi == GEMM_EPI_RESID_F32) {  // C is the fp32 accumulator
      ga.resid = static_cast<float*>(C);
      ga.ldr = ldc;
      ga.C = nullptr;
    }
    ga.a_mn = a_mn;
    ga.b_mn = b_mn;
    gemm_bf16(ga, s);
  };
  const int ACC = GEMM_EPI_RESID_F32;

  // ---- LM head (each rank's slice) and final norm (each rank's tokens) ------
  for (int r = 0; r < NLOC; ++r) {
    RankCtx& R = ranks_[r];
    if (R.lm_n == 0) continue;
    RW& w = rw[r];
    lmhead_dual_dlogits(lm_rows(R, 0), W.lm_head, lm_rows(R, ref_slot), Wr.lm_head, R.lm_n, V, d,
                        R.lm_idx.as<int32_t>(), coef_f + R.lm_lo, kw, kl_f + R.lm_lo, w.lsep,
                        w.lser, w.Gl, V, s);
    gemm_mn(w.Gl, V, 0, W.lm_head, d, 1, w.dxs, d, R.lm_n, d, V, GEMM_EPI_STORE_F32);
    gemm_mn(w.Gl, V, 1, lm_rows(R, 0), d, 1, grads_.lm_head, d, V, d, R.lm_n, ACC);
  }
  // the slices' dX rows back to the ranks owning the tokens (owner p's rows
  // land in its dxs buffer: a virtual rank's workspace or a peer's landing)
  auto dxs_dst = [&](int p) -> float* { return mesh_ ? mesh_->dxs(p) : rw[p].dxs_own; };
  if (mesh_) mesh_->barrier(s);  // every owner has consumed the previous group's rows
  for (int r = 0; r < NLOC; ++r) {
    const RankCtx& R = ranks_[r];
    for (int p = 0; p < K; ++p) {
      const long lo = std::max<long>(sc_lo[p], R.lm_lo);
      const long hi = std::min<long>(sc_lo[p] + n_sc[p], R.lm_lo + R.lm_n);
      if (hi <= lo) continue;
      MRSP_CUDA(cudaMemcpyAsync(dxs_dst(p) + (lo - sc_lo[p]) * d, rw[r].dxs + (lo - R.lm_lo) * d,
                                static_cast<size_t>(hi - lo) * d * 4, cudaMemcpyDeviceToDevice, s));
    }
  }
  if (mesh_) mesh_->barrier(s);  // every owner's rows have landed
  for (int r = 0; r < NLOC; ++r) {
    RankCtx& R = ranks_[r];
    RW& w = rw[r];
    const int n = static_cast<int>(R.e - R.b);
    MRSP_CUDA(cudaMemsetAsync(w.dh, 0, static_cast<size_t>(n) * d * 4, s));
    rmsnorm_bwd(R.h.as<float>(), d, W.final_norm, w.dxs_own, d, w.dh, d, R.n_scored, d, c.rms_eps,
                R.scored_idx.as<int32_t>(), grads_.final_norm, w.ws, s);
    negate_i32(R.pos.as<int>(), w.negpos, n, s);
  }

  // ---- decoder layers, last to first ----------------------------------------
  const float scale = 1.0f / std::sqrt(128.0f);
  for (int l = NL - 1; l >= 0; --l) {
    const LlmLayerW& Lw = W.layers[l];
    LlmLayerW& Lg = grads_.layers[l];
    // (1) recompute the layer's attention input: RMSNorm, QKV + RoPE routed to
    // the head shards (the forward's fused epilogue), attention with its lse
    // (unless the policy pass kept O and lse)
    for (int r = 0; r < NLOC; ++r) {
      RankCtx& R = ranks_[r];
      const int n = static_cast<int>(R.e - R.b);
      if (n <= 0) continue;
      const float* h_in = stash_bufs_[r].as<float>() + static_cast<size_t>(l) * n * d;
      rmsnorm(h_in, d, Lw.attn_norm, rw[r].xn1, d, n, d, c.rms_eps, nullptr, s);
      GemmArgs ga{rw[r].xn1, Lw.wqkv, nullptr, n, Cqkv, d, d, d, 0, GEMM_EPI_QKV_SCATTER, Lw.bqkv,
                  nullptr, 0};
      ga.pos = R.pos.as<int>();
      ga.inv_freq = d_inv_freq_;
      ga.n_rope_blocks = nq + nkv;
      ga.row0 = K == 1 ? 0 : R.b;
      ga.route = d_route_;
      ga.peer_base = d_peer_base_;
      ga.peer_ld = d_peer_ld_;
      ga.row_blocks = static_cast<int>((Ltot + ATTN_ROW_BLOCK - 1) / ATTN_ROW_BLOCK);
      gemm_bf16(ga, s);
    }
    if (mesh_) mesh_->barrier(s);  // every rank's head blocks have landed
    for (int r = 0; r < NLOC && !keep_attn; ++r) {
      RankCtx& R = ranks_[r];
      const int nqr = R.hs.nq();
      if (nqr == 0) continue;
      if (K == 1) {
        AttnParams ap{R.qkv.p, Cqkv, 0, R.qkv.p, Cqkv, nq * 128, R.qkv.p, Cqkv, (nq + nkv) * 128,
                      R.ol.p, Cq, 0, static_cast<int>(Ltot), nq, nq / nkv, scale,
                      ATTN_CAUSAL_PREFIX, static_cast<int>(g.Lp), g.Lmax, 0};
        ap.lse = rw[r].stat_lse;
        ap.lse_ld = rw[r].ld_stat;
        attention_fwd(ap, s);
      } else {
        // the forward's attention: head shard in, each O row stored straight
        // into its token owner's sequence shard (fused heads -> sequence)
        const int Cr = (nqr + 2 * R.hs.nkv()) * 128;
        void* qh = qh_dst(R.g);
        AttnParams ap{qh, Cr, 0, qh, Cr, nqr * 128, qh, Cr, (nqr + R.hs.nkv()) * 128,
                      nullptr, nqr * 128, 0, static_cast<int>(Ltot), nqr, R.hs.q_per_kv, scale,
                      ATTN_CAUSAL_PREFIX, static_cast<int>(g.Lp), g.Lmax, 0};
        ap.n_dst = K;
        for (int p = 0; p < K; ++p) {
          ap.dst_bounds[p] = token_b_[p];
          ap.dst_base[p] = ol_dst(p);
        }
        ap.dst_bounds[K] = token_e_[K - 1];
        ap.dst_ld = Cq;
        ap.dst_col0 = R.hs.q_lo * 128;
        ap.row_parts = R.hs.rparts;
        ap.row_part = R.hs.rpart;
        ap.lse = rw[r].stat_lse;
        ap.lse_ld = rw[r].ld_stat;
        attention_fwd(ap, s);
      }
    }
    if (mesh_) mesh_->barrier(s);  // every rank's O rows have landed
    // (2) per sequence shard: O projection, MLP recompute, MLP backward, the
    // post-attention RMSNorm backward, dO
    for (int r = 0; r < NLOC; ++r) {
      RankCtx& R = ranks_[r];
      RW& w = rw[r];
      const int n = static_cast<int>(R.e - R.b);
      if (n <= 0) continue;
      const size_t nd = static_cast<size_t>(n) * d;
      bf16* ol = keep_attn ? o_kept(r, l) : static_cast<bf16*>(ol_dst(R.g));
      const float* h_in = stash_bufs_[r].as<float>() + static_cast<size_t>(l) * nd;
      MRSP_CUDA(cudaMemcpyAsync(w.hm, h_in, nd * 4, cudaMemcpyDeviceToDevice, s));
      gemm_bf16({ol, Lw.wo, nullptr, n, d, Cq, Cq, Cq, 0, GEMM_EPI_RESID_F32, nullptr, w.hm, d}, s);
      rmsnorm(w.hm, d, Lw.mlp_norm, R.xn.as<bf16>(), d, n, d, c.rms_eps, nullptr, s);
      cast_f32_bf16(w.dh, d, w.dhb, d, n, d, s);
      gemm_mn(w.dhb, d, 0, Lw.wdown, mlp, 1, w.dact, mlp, n, mlp, d, GEMM_EPI_STORE_BF16);
      {
        GemmArgs ga{R.xn.p, Lw.wgu, w.dgu, n, 2 * mlp, d, d, d, 2 * mlp, GEMM_EPI_SWIGLU_BWD,
                    nullptr, nullptr, 0};
        ga.aux = w.dact;
        ga.ld_aux = mlp;
        ga.aux_out = R.act.p;
        ga.ld_aux_out = mlp;
        gemm_bf16(ga, s);
      }
      gemm_mn(w.dhb, d, 1, R.act.p, mlp, 1, Lg.wdown, mlp, d, mlp, n, ACC);
      gemm_mn(w.dgu, 2 * mlp, 1, R.xn.p, d, 1, Lg.wgu, d, 2 * mlp, d, n, ACC);
      gemm_mn(w.dgu, 2 * mlp, 0, Lw.wgu, d, 1, w.dx, d, n, d, 2 * mlp, GEMM_EPI_STORE_F32);
      rmsnorm_bwd(w.hm, d, Lw.mlp_norm, w.dx, d, w.dh, d, n, d, c.rms_eps, nullptr, Lg.mlp_norm,
                  w.ws, s);
      cast_f32_bf16(w.dh, d, w.dhb, d, n, d, s);
      gemm_mn(w.dhb, d, 0, Lw.wo, Cq, 1, w.dO, Cq, n, Cq, d, GEMM_EPI_STORE_BF16);
      gemm_mn(w.dhb, d, 1, ol, Cq, 1, Lg.wo, Cq, d, Cq, n, ACC);
      if (K > 1) attention_rowdot(w.dO, Cq, ol, Cq, n, nq, w.dseq, w.ld_dseq, s);
    }
    if (K > 1) {  // sequence -> heads: dO columns and row dots to the head owners
      for (int r = 0; r < NLOC; ++r) {
        const RankCtx& R = ranks_[r];
        route_seq_to_heads(ra, R.b, R.e, rw[r].dO, Cq, rw[r].dseq, rw[r].ld_dseq, s);
      }
      if (mesh_) mesh_->barrier(s);
    }
    // (3) attention backward on the head shards
    for (int r = 0; r < NLOC; ++r) {
      RankCtx& R = ranks_[r];
      const int nqr = R.hs.nq();
      if (nqr == 0) continue;
      Prof pa(*this, P_BWD_ATTN);
      float* lse = keep_attn ? lse_kept(r, l) : rw[r].stat_lse;
      if (K == 1) {
        AttnBwdParams bp{R.qkv.p, Cqkv, 0, nq * 128, (nq + nkv) * 128,
                         keep_attn ? static_cast<void*>(o_kept(r, l)) : R.ol.p, Cq, rw[r].dO, Cq,
                         lse, rw[r].stat_D, rw[r].ld_stat, rw[r].dqkv, Cqkv,
                         static_cast<int>(Ltot), nq, nq / nkv, scale, static_cast<int>(g.Lp), g.Lmax};
        attention_bwd(bp, s);
      } else {
        const int Cr = (nqr + 2 * R.hs.nkv()) * 128;
        AttnBwdParams bp{qh_dst(R.g), Cr, 0, nqr * 128, (nqr + R.hs.nkv()) * 128, nullptr, nqr * 128,
                         rw[r].doh, nqr * 128, lse, rw[r].stat_D, rw[r].ld_stat,
                         rw[r].dqkvh, Cr, static_cast<int>(Ltot), nqr, R.hs.q_per_kv, scale,
                         static_cast<int>(g.Lp), g.Lmax};
        bp.d_given = 1;
        bp.row_parts = R.hs.rparts;
        bp.row_part = R.hs.rpart;
        bp.dkv32 = rw[r].dkv32;
        bp.ld_dkv32 = 2 * R.hs.nkv() * 128;
        attention_bwd(bp, s);
      }
    }
    if (K > 1) {  // heads -> sequence: dq rows, dk / dv rows (or partials) to the owners
      for (int r = 0; r < NLOC; ++r) {
        const RankCtx& R = ranks_[r];
        if (R.hs.nq() == 0) continue;
        route_heads_to_seq(ra, R.g, rw[r].dqkvh, (R.hs.nq() + 2 * R.hs.nkv()) * 128, rw[r].dkv32,
                           2 * R.hs.nkv() * 128, s);
      }
      if (mesh_) mesh_->barrier(s);
      if (m_kv > 1)  // kv heads shared by m ranks: their partial dk / dv summed in slot order
        for (int r = 0; r < NLOC; ++r) {
          const RankCtx& R = ranks_[r];
          kv_partial_sum(rw[r].slots, m_kv, R.e - R.b, nkv, rw[r].dqkv, nq, s);
        }
    }
    // (4) per sequence shard: RoPE backward, QKV bias / weight gradients, dX,
    // the input RMSNorm backward
    for (int r = 0; r < NLOC; ++r) {
      RankCtx& R = ranks_[r];
      RW& w = rw[r];
      const int n = static_cast<int>(R.e - R.b);
      if (n <= 0) continue;
      const float* h_in = stash_bufs_[r].as<float>() + static_cast<size_t>(l) * n * d;
      rope(w.dqkv, Cqkv, 0, nq + nkv, w.negpos, n, s);  // transpose rotation of the q / k heads
      colsum_bf16(w.dqkv, Cqkv, n, Cqkv, Lg.bqkv, w.ws, s);
      gemm_mn(w.dqkv, Cqkv, 1, w.xn1, d, 1, Lg.wqkv, d, Cqkv, d, n, ACC);
      gemm_mn(w.dqkv, Cqkv, 0, Lw.wqkv, d, 1, w.dx, d, n, d, Cqkv, GEMM_EPI_STORE_F32);
      rmsnorm_bwd(h_in, d, Lw.attn_norm, w.dx, d, w.dh, d, n, d, c.rms_eps, nullptr, Lg.attn_norm,
                  w.ws, s);
    }
  }
  }  // Prof P_BACKWARD

  // ---- text embeddings: dE[tok] += dh at the token's positions, per shard ---
  std::vector<int> blob_all;
  {
    float* dE = reinterpret_cast<float*>(grads_.embed);
    std::vector<std::pair<int, long>> tp;  // (token, global position) of the text positions
    for (int i = 0; i < n_q; ++i) tp.emplace_back(question[i], g.n_frame_tok + i);
    for (int r = 0; r < G; ++r)
      for (int j = 0; j < lengths[r]; ++j)
        tp.emplace_back(j == 0 ? 1 /* Vocab::kEos */ : resp[static_cast<size_t>(r) * Lmax + j - 1],
                        g.Lp + static_cast<long>(r) * Lmax + j);
    for (int r = 0; r < NLOC; ++r) {
      RankCtx& R = ranks_[r];
      std::map<int, std::vector<int>> at;  // token -> ascending local rows
      for (const auto& t : tp)
        if (t.second >= R.b && t.second < R.e) at[t.first].push_back(static_cast<int>(t.second - R.b));
      if (at.empty()) continue;
      std::vector<int> seg_tok, seg_off{0}, positions;
      for (auto& kv : at) {
        seg_tok.push_back(kv.first);
        positions.insert(positions.end(), kv.second.begin(), kv.second.end());
        seg_off.push_back(static_cast<int>(positions.size()));
      }
      const int n_seg = static_cast<int>(seg_tok.size());
      std::vector<int> blob;
      blob.insert(blob.end(), seg_tok.begin(), seg_tok.end());
      blob.insert(blob.end(), seg_off.begin(), seg_off.end());
      blob.insert(blob.end(), positions.begin(), positions.end());
      int* dblob = static_cast<int*>(R.send.ensure(blob.size() * 4 + 16));
      MRSP_CUDA(cudaMemcpyAsync(dblob, blob.data(), blob.size() * 4, cudaMemcpyHostToDevice, s));
      embed_grad(rw[r].dh, d, dblob, dblob + n_seg, dblob + 2 * n_seg + 1, n_seg, dE, s);
      MRSP_CUDA(cudaStreamSynchronize(s));  // the host blob goes out of scope
    }
  }
  // ---- across processes: every rank's weight gradients summed in rank order
  // (chunked through the peer mesh's staging slots; identical on every rank)
  if (mesh_) {
    float* gr = static_cast<float*>(grad_buf_.p);
    const long total = static_cast<long>(grad_bytes / 4), chunk = mesh_->caps().red_floats;
    const int me = ranks_[0].g;
    for (long off = 0; off < total; off += chunk) {
      const long n = std::min(chunk, total - off);
      mesh_->barrier(s);  // every rank has summed the previous chunk's slots
      for (int p = 0; p < K; ++p)
        MRSP_CUDA(cudaMemcpyAsync(mesh_->red(p) + static_cast<size_t>(me) * chunk, gr + off,
                                  static_cast<size_t>(n) * 4, cudaMemcpyDeviceToDevice, s));
      mesh_->barrier(s);  // every rank's chunk has landed
      slot_sum_f32(mesh_->red(me), K, chunk, n, gr + off, s);
    }
    mesh_->barrier(s);
  }
  std::vector<float> lp_host(S);
  MRSP_CUDA(cudaMemcpyAsync(lp_host.data(), lp_f, static_cast<size_t>(S) * 4, cudaMemcpyDeviceToHost, s));
  if (mode == 0)
    MRSP_CUDA(cudaMemcpyAsync(stats4, d_stats, 4 * sizeof(double), cudaMemcpyDeviceToHost, s));
  MRSP_CUDA(cudaStreamSynchronize(s));
  if (mode == 1) {  // loss = mean -log pi(y), summed in group order in double
    double loss = 0.0;
    for (int i = 0; i < S; ++i) loss -= lp_host[i];
    stats4[0] = loss / S;
    stats4[1] = stats4[2] = 0.0;
    stats4[3] = S;
  }
  if (lp_out) std::copy(lp_host.begin(), lp_host.end(), lp_out);
  prof_collect();
  have_grads_ = true;
}

}  // namespace mrsp
