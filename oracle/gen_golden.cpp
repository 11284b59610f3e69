// gen_golden.cpp — generates tests/golden/ref_toy.json by running the
// REFERENCE's own code (compiled from /root/reference/proj/src by
// oracle/Makefile into oracle/_ref/). TEST INFRASTRUCTURE ONLY.
//
// The fixture pins oracle/mrsp_oracle.c (the CPU restatement) and the B200
// toy path to the reference bit for bit: shard plans (engine.cpp:15-29), pad
// rows (engine.cpp:31-50), synthetic frames (mmseq.cpp:58-72), encoder and
// policy init (policy.cpp:12-34, :56-61), encode_frame (policy.cpp:36-47),
// serial_prefill/step_logits (engine.cpp:59-71, policy.cpp:85-119),
// log_softmax (common.hpp:95-104), cache/bench counters (engine.cpp:155-283),
// GRPO stats (grpo.cpp:68-108) and the analytic GRPO / SFT gradients
// (grpo.cpp:122-223, policy.cpp:195-260).
#include <cstdio>
#include <fstream>
#include <iostream>

#include "json.hpp"
#include "lvrl/engine.hpp"
#include "lvrl/grpo.hpp"

using namespace lvrl;
using json = nlohmann::ordered_json;

int main(int argc, char** argv) {
  const char* path = argc > 1 ? argv[1] : "ref_toy.json";
  json j;

  // plan_shards hand examples + the big token plans of the BASELINE configs.
  json plans = json::array();
  for (auto [n, k] : std::vector<std::pair<std::size_t, int>>{
           {10, 3}, {2, 4}, {0, 3}, {7, 1}, {131104, 8}, {65568, 4}, {139301, 8}, {16421 + 8 * 1024, 2}}) {
    auto p = mrsp::plan_shards(n, k);
    json r = json::array();
    for (auto [b, e] : p.ranges) r.push_back({b, e});
    plans.push_back({{"n", n}, {"k", k}, {"ranges", r}});
  }
  j["plan_shards"] = plans;

  {
    std::vector<std::vector<TokenId>> rows = {{5, 6, 7}, {8}, {9, 10, 11, 12, 13}, {}};
    auto b = mrsp::pad_batch(rows);
    j["pad_batch"] = {{"rows_in", rows}, {"rows", b.rows}, {"lengths", b.lengths},
                      {"max_len", b.max_len}};
  }

  {
    Rng r = Rng::substream(7, "video");
    j["substream_7_video_first"] = std::to_string(r.next_u64());
    auto v = mmseq::gen_video(7, 2, 4);
    json fr = json::array();
    for (auto& f : v.frames) fr.push_back(f.features);
    j["gen_video_7_2_4"] = {{"id", v.id}, {"frames", fr}};
  }

  // Encoder + encode of a small video.
  {
    auto enc = policy::EncoderParams::generate(1234, 8, 16);
    auto v = mmseq::gen_video(9, 5, 16);
    auto e = mrsp::serial_encode(enc, v);
    j["encoder_1234_8_16"] = enc.w;
    j["encode_v9f5"] = e;
  }
  // A bench-shaped encode (d 128, p 256) for 3 frames.
  {
    auto enc = policy::EncoderParams::generate(1234, 128, 256);
    auto v = mmseq::gen_video(1234 + 64 * 100, 3, 256);
    j["encode_bench_shape"] = mrsp::serial_encode(enc, v);
  }

  // Policy init + step_logits + log_softmax.
  {
    policy::PolicyDims dims{32, 8, 12, 16};
    auto params = policy::PolicyParams::random(dims, 4, 0.4);
    j["policy_32_8_12_seed4"] = params.theta;
    Vec ctx(dims.d, 0.1);
    auto logits = policy::step_logits(params, ctx, mmseq::Vocab::kEos);
    j["step_logits_ctx01_eos"] = logits;
    j["log_softmax_of_that"] = log_softmax(logits);

    // serial_prefill on a ragged batch (one empty row included).
    std::vector<std::vector<TokenId>> rows = {{5, 6, 7, 30}, {9}, {}, {11, 12, 13, 14, 15, 16}};
    auto batch = mrsp::pad_batch(rows);
    std::vector<Vec> contexts;
    Rng rng(77);
    for (std::size_t i = 0; i < rows.size(); ++i) {
      Vec c(dims.d);
      for (double& x : c) x = rng.normal();
      contexts.push_back(c);
    }
    auto out = mrsp::serial_prefill(params, contexts, batch);
    json o = json::array();
    for (auto& r : out) o.push_back(r);
    j["prefill"] = {{"rows", rows}, {"contexts", contexts}, {"logits", o}};

    // context_vector over an encoded video + question template {10,11,12}.
    auto enc = policy::EncoderParams::generate(2, 8, 16);
    auto v = mmseq::gen_video(3, 4, 16);
    mmseq::MultimodalSequence seq;
    seq.frame_embeddings = mrsp::serial_encode(enc, v);
    seq.text_tokens = {10, 11, 12};
    j["context_vector"] = policy::context_vector(seq, params);
  }

  // Cache counter script (test_engine.cpp:189-221 shape) on the reference engine.
  {
    auto enc = policy::EncoderParams::generate(7, 8, 16);
    mrsp::WorkerGroup group(2, enc);
    mrsp::EmbeddingCache cache;
    auto a = mmseq::gen_video(1, 6, 16), b = mmseq::gen_video(2, 6, 16);
    auto plan = mrsp::plan_shards(6, 2);
    json script = json::array();
    for (auto* v : {&a, &a, &b, &a, &b}) {
      bool hit = cache.get_or_encode(group, *v, plan).second;
      script.push_back({{"video", v->id}, {"hit", hit},
                        {"invocations", group.stats().encoder_invocations.load()},
                        {"misses", group.stats().cache_misses.load()},
                        {"hits", group.stats().cache_hits.load()},
                        {"gather_bytes", group.stats().gather_bytes.load()}});
    }
    j["cache_script"] = script;
  }

  // GRPO token terms (grpo.cpp:68-108) on a sampled group: per-token inputs
  // from the public API + the reference's own GroupStats, exact and sampled KL.
  {
    policy::PolicyDims dims{32, 8, 12, 16};
    auto theta = policy::PolicyParams::random(dims, 17, 0.4);
    auto ref = policy::PolicyParams::random(dims, 18, 0.4);
    auto enc = policy::EncoderParams::generate(1, 8, 16);
    auto video = mmseq::gen_video(3, 8, 16);
    auto sample = mmseq::gen_task(video, mmseq::TaskFamily::ArgmaxChannel);
    auto seq = mmseq::build_sequence(mrsp::serial_encode(enc, video), sample);
    auto theta_old = policy::PolicyParams::random(dims, 19, 0.4);  // ratios != 1
    Rng rng(6);
    grpo::RolloutGroup group;
    Vec rewards;
    for (int i = 0; i < 6; ++i) {
      auto r = policy::sample_rollout(theta_old, seq, 1.0, 12, rng);
      rewards.push_back(rng.uniform());
      group.rollouts.push_back(std::move(r));
    }
    group.advantages = grpo::compute_advantages(rewards, 1e-8);
    json rolls = json::array();
    for (const auto& r : group.rollouts) {
      rolls.push_back({{"tokens", r.tokens},
                       {"old_logprobs", r.old_logprobs},
                       {"logprobs", policy::sequence_logprobs(theta, seq, r.tokens)},
                       {"ref_logprobs", policy::sequence_logprobs(ref, seq, r.tokens)},
                       {"kl", policy::kl_per_position(theta, ref, seq, r.tokens)}});
    }
    grpo::GrpoConfig cfg;
    grpo::GroupStats exact, sampled;
    grpo::grpo_objective(group, theta, ref, seq, cfg, &exact);
    cfg.sampled_kl = true;
    grpo::grpo_objective(group, theta, ref, seq, cfg, &sampled);
    auto st = [](const grpo::GroupStats& g) {
      return json{{"objective", g.objective}, {"mean_kl", g.mean_kl},
                  {"clip_fraction", g.clip_fraction}, {"token_count", g.token_count}};
    };
    j["grpo"] = {{"rollouts", rolls}, {"advantages", group.advantages.values},
                 {"clip_eps", cfg.clip_eps}, {"kl_beta", cfg.kl_beta},
                 {"stats_exact_kl", st(exact)}, {"stats_sampled_kl", st(sampled)}};

    // Backward (grpo.cpp:122-223, policy.cpp:195-260): the reference's exact
    // analytic gradients on the same group and sequence — exact KL, sampled
    // (k3) KL, no KL — and SFT loss + gradient on the sample's SFT target.
    grpo::GroupStats g_exact, g_sampled, g_nokl;
    cfg.sampled_kl = false;
    Vec grad_exact = grpo::grpo_gradient(group, theta, ref, seq, cfg, &g_exact);
    cfg.sampled_kl = true;
    Vec grad_sampled = grpo::grpo_gradient(group, theta, ref, seq, cfg, &g_sampled);
    cfg.sampled_kl = false;
    cfg.kl_beta = 0.0;
    Vec grad_nokl = grpo::grpo_gradient(group, theta, ref, seq, cfg, &g_nokl);
    auto target = grpo::sft_target(sample);
    auto [sft_loss, sft_grad] = grpo::sft_loss_and_grad(theta, seq, target);
    j["backward"] = {{"theta", theta.theta}, {"ref", ref.theta},
                     {"frame_embeddings", seq.frame_embeddings}, {"text_tokens", seq.text_tokens},
                     {"clip_eps", 0.2}, {"kl_beta", 0.04},
                     {"grad_exact_kl", grad_exact}, {"stats_exact_kl", st(g_exact)},
                     {"grad_sampled_kl", grad_sampled}, {"stats_sampled_kl", st(g_sampled)},
                     {"grad_no_kl", grad_nokl}, {"stats_no_kl", st(g_nokl)},
                     {"sft_target", target}, {"sft_loss", sft_loss}, {"sft_grad", sft_grad}};
  }

  std::ofstream(path) << j.dump(1) << "\n";
  std::cout << "wrote " << path << "\n";
  return 0;
}
