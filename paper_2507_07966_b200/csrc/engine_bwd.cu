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
//                RoPE, attention (with its log-sum-exp), O projection, RMSNorm;
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
  MRSP_REQUIRE(k_ == 1 && !mesh_ && !nccl_, MRSP_INVALID_ARGUMENT,
               "grpo_backward: sequence parallel backward is not built; use an SP = 1 engine");
  MRSP_REQUIRE(has_ref_ || kl_beta == 0.0, MRSP_INVALID_ARGUMENT,
               "grpo_backward: the KL term needs a separate reference model");
  MRSP_REQUIRE(old_lp && adv && stats4, MRSP_INVALID_ARGUMENT, "grpo_backward: null argument");
  MRSP_REQUIRE(clip_eps >= 0.0, MRSP_INVALID_ARGUMENT, "grpo_backward: clip_eps < 0");
  std::lock_guard<std::mutex> run(run_mu_);
  const auto& c = cfg_;
  const int d = c.dim, nq = c.n_q_heads, nkv = c.n_kv_heads, mlp = c.mlp, V = c.vocab;
  const int Cqkv = (nq + 2 * nkv) * 128, Cq = nq * 128, NL = c.layers;
  MRSP_REQUIRE(d % 8 == 0 && mlp % 128 == 0 && V % 8 == 0, MRSP_INVALID_ARGUMENT,
               "grpo_backward: unsupported model geometry");
  cudaStream_t s = stream_;
  prepare_group(emb, question, n_q, resp, lengths, G, Lmax);
  const GroupState& g = grp_;
  RankCtx& R = ranks_[0];
  const int n = static_cast<int>(R.e - R.b);
  const int S = R.n_scored;
  MRSP_REQUIRE(S == g.total_scored && S >= 1, MRSP_INVALID_ARGUMENT,
               "grpo_backward: the group has no scored token");

  // ---- gradient storage: fp32 in the engine's weight layout ----------------
  if (!grad_buf_.p) {
    size_t tot = 0;
    auto add = [&](size_t elems) { tot += (elems * 4 + 255) & ~size_t(255); };
    add(static_cast<size_t>(V) * d);
    for (int l = 0; l < NL; ++l) {
      add(d); add(static_cast<size_t>(Cqkv) * d); add(Cqkv); add(static_cast<size_t>(d) * Cq);
      add(d); add(static_cast<size_t>(2) * mlp * d); add(static_cast<size_t>(d) * mlp);
    }
    add(d);
    add(static_cast<size_t>(V) * d);
    grad_buf_.ensure(tot);
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

  // ---- workspaces ------------------------------------------------------------
  const size_t nd = static_cast<size_t>(n) * d;
  const int ld_stat = (n + 3) / 4 * 4;
  const int ldg = V;
  const size_t ws_norm = rmsnorm_bwd_workspace_bytes(std::max(n, S), d);
  const size_t ws_col = colsum_workspace_bytes(n, Cqkv);
  const size_t dual_ws = lmhead_dual_workspace_bytes(S, V);
  {
    size_t tot = 0;
    auto add = [&](size_t bytes) { tot += (bytes + 255) & ~size_t(255); };
    add(nd * 4 * 3);                                   // hm, dh, dx
    add(nd * 2 * 2);                                   // dhb, xn1
    add(static_cast<size_t>(n) * mlp * 2);             // dact
    add(static_cast<size_t>(n) * 2 * mlp * 2);         // dgu
    add(static_cast<size_t>(n) * Cq * 2);              // dO
    add(static_cast<size_t>(n) * Cqkv * 2);            // dqkv
    add(static_cast<size_t>(nq) * ld_stat * 4 * 2);    // lse, D
    add(static_cast<size_t>(n) * 4);                   // -pos
    add(static_cast<size_t>(S) * ldg * 2);             // G
    add(static_cast<size_t>(S) * d * 4);               // dxs
    add(static_cast<size_t>(S) * 4 * 8);               // lp, lp_ref, kl, lse_p, lse_r, coef, old
    add(static_cast<size_t>(G) * 4 * 2 + 64);          // adv, lengths, stats
    add(std::max(ws_norm, ws_col));
    add(dual_ws);
    bwd_ws_.ensure(tot);
  }
  Carve cv{static_cast<uint8_t*>(bwd_ws_.p)};
  float* hm = cv.take<float>(nd);
  float* dh = cv.take<float>(nd);
  float* dx = cv.take<float>(nd);
  bf16* dhb = cv.take<bf16>(nd);
  bf16* xn1 = cv.take<bf16>(nd);
  bf16* dact = cv.take<bf16>(static_cast<size_t>(n) * mlp);
  bf16* dgu = cv.take<bf16>(static_cast<size_t>(n) * 2 * mlp);
  bf16* dO = cv.take<bf16>(static_cast<size_t>(n) * Cq);
  bf16* dqkv = cv.take<bf16>(static_cast<size_t>(n) * Cqkv);
  float* lse = cv.take<float>(static_cast<size_t>(nq) * ld_stat);
  float* Dst = cv.take<float>(static_cast<size_t>(nq) * ld_stat);
  int* negpos = cv.take<int>(n);
  bf16* Gl = cv.take<bf16>(static_cast<size_t>(S) * ldg);
  float* dxs = cv.take<float>(static_cast<size_t>(S) * d);
  float* lp = cv.take<float>(S);
  float* lp_ref = cv.take<float>(S);
  float* kl = cv.take<float>(S);
  float* lse_p = cv.take<float>(S);
  float* lse_r = cv.take<float>(S);
  float* coef = cv.take<float>(S);
  float* d_old = cv.take<float>(S);
  float* d_adv = cv.take<float>(G);
  double* d_stats = cv.take<double>(4);
  void* ws = cv.take<uint8_t>(std::max(ws_norm, ws_col));
  void* dws = cv.take<uint8_t>(dual_ws);
  stash_buf_.ensure(static_cast<size_t>(NL) * nd * 4);

  // ---- forward: reference pass, then the policy pass keeping layer inputs --
  run_pass(emb, 1, 1);  // R.xs2 = reference final-norm rows
  stash_ = stash_buf_.as<float>();
  try {
    run_pass(emb, 0, 0);  // R.xs = policy final-norm rows; R.h = h_L
  } catch (...) {
    stash_ = nullptr;
    throw;
  }
  stash_ = nullptr;
  const LlmW& W = llm_[0];
  const LlmW& Wr = llm_[1];
  {
    Prof pl(*this, P_LMHEAD);
    lmhead_dual_logprob_kl_lse(R.xs.p, W.lm_head, R.xs2.p, Wr.lm_head, S, V, d,
                               R.lm_idx.as<int32_t>(), lp, lp_ref, kl, lse_p, lse_r, dws, dual_ws, s);
  }
  MRSP_CUDA(cudaMemcpyAsync(d_old, old_lp, static_cast<size_t>(S) * 4, cudaMemcpyHostToDevice, s));
  MRSP_CUDA(cudaMemcpyAsync(d_adv, adv, static_cast<size_t>(G) * 4, cudaMemcpyHostToDevice, s));
  grpo_stats(lp, d_old, lp_ref, kl, d_adv, g.d_len, G, clip_eps, kl_beta, sampled_kl, d_stats, s);
  {
  Prof pb(*this, P_BACKWARD);
  grpo_token_coeffs(lp, d_old, lp_ref, d_adv, g.d_len, G, S, clip_eps, kl_beta, sampled_kl, coef, s);
  const float kw = (sampled_kl || kl_beta == 0.0) ? 0.f : static_cast<float>(-kl_beta / S);

  // ---- LM head and final norm -------------------------------------------------
  lmhead_dual_dlogits(R.xs.p, W.lm_head, R.xs2.p, Wr.lm_head, S, V, d, R.lm_idx.as<int32_t>(),
                      coef, kw, kl, lse_p, lse_r, Gl, ldg, s);
  auto gemm_mn = [&](const void* A, int lda, int a_mn, const void* B, int ldb, int b_mn, void* C,
                     int ldc, int M, int N, int K, int epi, float* resid = nullptr, int ldr = 0) {
    GemmArgs ga{A, B, C, M, N, K, lda, ldb, ldc, epi, nullptr, resid, ldr};
    ga.a_mn = a_mn;
    ga.b_mn = b_mn;
    gemm_bf16(ga, s);
  };
  // dX_s = G . W_lm  (W_lm [V][d] read as the MN-major B of an [S x d x V] GEMM)
  gemm_mn(Gl, ldg, 0, W.lm_head, d, 1, dxs, d, S, d, V, GEMM_EPI_STORE_F32);
  // dW_lm = G^T . X_s
  gemm_mn(Gl, ldg, 1, R.xs.p, d, 1, grads_.lm_head, d, V, d, S, GEMM_EPI_STORE_F32);
  MRSP_CUDA(cudaMemsetAsync(dh, 0, nd * 4, s));
  rmsnorm_bwd(R.h.as<float>(), d, W.final_norm, dxs, d, dh, d, S, d, c.rms_eps,
              R.scored_idx.as<int32_t>(), grads_.final_norm, ws, s);

  // ---- decoder layers, last to first ----------------------------------------
  negate_i32(R.pos.as<int>(), negpos, n, s);
  const float scale = 1.0f / std::sqrt(128.0f);
  for (int l = NL - 1; l >= 0; --l) {
    const LlmLayerW& Lw = W.layers[l];
    LlmLayerW& Lg = grads_.layers[l];
    const float* h_in = stash_buf_.as<float>() + static_cast<size_t>(l) * nd;
    // recompute the layer's forward (the same kernels as run_pass at SP = 1)
    rmsnorm(h_in, d, Lw.attn_norm, xn1, d, n, d, c.rms_eps, nullptr, s);
    {
      GemmArgs ga{xn1, Lw.wqkv, nullptr, n, Cqkv, d, d, d, 0, GEMM_EPI_QKV_SCATTER, Lw.bqkv,
                  nullptr, 0};
      ga.pos = R.pos.as<int>();
      ga.inv_freq = d_inv_freq_;
      ga.n_rope_blocks = nq + nkv;
      ga.row0 = 0;
      ga.route = d_route_;
      ga.peer_base = d_peer_base_;
      ga.peer_ld = d_peer_ld_;
      ga.row_blocks = static_cast<int>((g.Ltot + ATTN_ROW_BLOCK - 1) / ATTN_ROW_BLOCK);
      gemm_bf16(ga, s);
    }
    {
      AttnParams ap{R.qkv.p, Cqkv, 0, R.qkv.p, Cqkv, nq * 128, R.qkv.p, Cqkv, (nq + nkv) * 128,
                    R.ol.p, Cq, 0, n, nq, nq / nkv, scale, ATTN_CAUSAL_PREFIX,
                    static_cast<int>(g.Lp), g.Lmax, 0};
      ap.lse = lse;
      ap.lse_ld = ld_stat;
      attention_fwd(ap, s);
    }
    MRSP_CUDA(cudaMemcpyAsync(hm, h_in, nd * 4, cudaMemcpyDeviceToDevice, s));
    gemm_bf16({R.ol.p, Lw.wo, nullptr, n, d, Cq, Cq, Cq, 0, GEMM_EPI_RESID_F32, nullptr, hm, d}, s);
    rmsnorm(hm, d, Lw.mlp_norm, R.xn.as<bf16>(), d, n, d, c.rms_eps, nullptr, s);
    // MLP backward
    cast_f32_bf16(dh, d, dhb, d, n, d, s);
    gemm_mn(dhb, d, 0, Lw.wdown, mlp, 1, dact, mlp, n, mlp, d, GEMM_EPI_STORE_BF16);
    {
      GemmArgs ga{R.xn.p, Lw.wgu, dgu, n, 2 * mlp, d, d, d, 2 * mlp, GEMM_EPI_SWIGLU_BWD, nullptr,
                  nullptr, 0};
      ga.aux = dact;
      ga.ld_aux = mlp;
      ga.aux_out = R.act.p;
      ga.ld_aux_out = mlp;
      gemm_bf16(ga, s);
    }
    gemm_mn(dhb, d, 1, R.act.p, mlp, 1, Lg.wdown, mlp, d, mlp, n, GEMM_EPI_STORE_F32);
    gemm_mn(dgu, 2 * mlp, 1, R.xn.p, d, 1, Lg.wgu, d, 2 * mlp, d, n, GEMM_EPI_STORE_F32);
    gemm_mn(dgu, 2 * mlp, 0, Lw.wgu, d, 1, dx, d, n, d, 2 * mlp, GEMM_EPI_STORE_F32);
    rmsnorm_bwd(hm, d, Lw.mlp_norm, dx, d, dh, d, n, d, c.rms_eps, nullptr, Lg.mlp_norm, ws, s);
    // attention backward
    cast_f32_bf16(dh, d, dhb, d, n, d, s);
    gemm_mn(dhb, d, 0, Lw.wo, Cq, 1, dO, Cq, n, Cq, d, GEMM_EPI_STORE_BF16);
    gemm_mn(dhb, d, 1, R.ol.p, Cq, 1, Lg.wo, Cq, d, Cq, n, GEMM_EPI_STORE_F32);
    {
      Prof pa(*this, P_BWD_ATTN);
      AttnBwdParams bp{R.qkv.p, Cqkv, 0, nq * 128, (nq + nkv) * 128, R.ol.p, Cq, dO, Cq, lse, Dst,
                       ld_stat, dqkv, Cqkv, n, nq, nq / nkv, scale, static_cast<int>(g.Lp), g.Lmax};
      attention_bwd(bp, s);
    }
    rope(dqkv, Cqkv, 0, nq + nkv, negpos, n, s);  // transpose rotation of the q / k heads
    colsum_bf16(dqkv, Cqkv, n, Cqkv, Lg.bqkv, ws, s);
    gemm_mn(dqkv, Cqkv, 1, xn1, d, 1, Lg.wqkv, d, Cqkv, d, n, GEMM_EPI_STORE_F32);
    gemm_mn(dqkv, Cqkv, 0, Lw.wqkv, d, 1, dx, d, n, d, Cqkv, GEMM_EPI_STORE_F32);
    rmsnorm_bwd(h_in, d, Lw.attn_norm, dx, d, dh, d, n, d, c.rms_eps, nullptr, Lg.attn_norm, ws, s);
  }
  }  // Prof P_BACKWARD

  // ---- text embeddings: dE[tok] = sum of dh at the token's positions ---------
  {
    std::map<int, std::vector<int>> at;  // token -> ascending positions (text, non-pad)
    for (int i = 0; i < n_q; ++i) at[question[i]].push_back(static_cast<int>(g.n_frame_tok) + i);
    for (int r = 0; r < G; ++r)
      for (int j = 0; j < lengths[r]; ++j) {
        const int tok = j == 0 ? 1 /* Vocab::kEos */ : resp[static_cast<size_t>(r) * Lmax + j - 1];
        at[tok].push_back(static_cast<int>(g.Lp + static_cast<long>(r) * Lmax + j));
      }
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
    float* dE = reinterpret_cast<float*>(grads_.embed);
    MRSP_CUDA(cudaMemsetAsync(dE, 0, static_cast<size_t>(V) * d * 4, s));
    embed_grad(dh, d, dblob, dblob + n_seg, dblob + 2 * n_seg + 1, n_seg, dE, s);
    MRSP_CUDA(cudaMemcpyAsync(stats4, d_stats, 4 * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (lp_out) MRSP_CUDA(cudaMemcpyAsync(lp_out, lp, static_cast<size_t>(S) * 4, cudaMemcpyDeviceToHost, s));
    MRSP_CUDA(cudaStreamSynchronize(s));  // host blob goes out of scope
  }
  prof_collect();
  have_grads_ = true;
}

}  // namespace mrsp
