// grpo_stats.cu — GRPO token terms over the engine's per-token outputs, the
// immediate consumer of the two prefill passes:
// evaluate_from_logits (grpo.cpp:68-108) given log pi_theta(y), log pi_old(y),
// log pi_ref(y) and the exact per-token KL from the fused dual LM head:
//   ratio = exp(lp - old); clipped = clamp(ratio, 1 - eps, 1 + eps)
//   seq_term_g = sum_t min(ratio A_g, clipped A_g);  policy = sum_g seq_term_g / len_g / G
//   clipped token iff (A > 0 && ratio > 1 + eps) || (A < 0 && ratio < 1 - eps)
//   kl_t = exact KL (sampled_kl = 0) or k3 = e^(lr) - 1 - lr, lr = lp_ref - lp
//   objective = policy - beta * mean_kl.
// fp64 arithmetic; one lane per rollout walks its tokens in order, then a
// fixed-order reduction — deterministic.
#include <cuda_runtime.h>

#include "backward.h"
#include "common.h"

namespace mrsp {
namespace {

__global__ void grpo_stats_kernel(const float* __restrict__ lp, const float* __restrict__ old_lp,
                                  const float* __restrict__ lp_ref, const float* __restrict__ kl,
                                  const float* __restrict__ adv, const int* __restrict__ lengths,
                                  int G, double clip_eps, double beta, int sampled,
                                  double* __restrict__ out) {
  __shared__ double s_pol[1024], s_kl[1024], s_clip[1024], s_n[1024];
  for (int g = threadIdx.x; g < G; g += blockDim.x) {
    long off = 0;
    for (int i = 0; i < g; ++i) off += lengths[i];
    const double A = adv[g];
    double seq = 0.0, kls = 0.0, ncl = 0.0;
    for (int t = 0; t < lengths[g]; ++t) {
      const double l = lp[off + t];
      const double ratio = exp(l - static_cast<double>(old_lp[off + t]));
      const double clipped = fmin(fmax(ratio, 1.0 - clip_eps), 1.0 + clip_eps);
      seq += fmin(ratio * A, clipped * A);
      if ((A > 0 && ratio > 1.0 + clip_eps) || (A < 0 && ratio < 1.0 - clip_eps)) ncl += 1.0;
      if (sampled) {
        const double lr = static_cast<double>(lp_ref[off + t]) - l;
        kls += exp(lr) - 1.0 - lr;
      } else {
        kls += kl[off + t];
      }
    }
    s_pol[g] = lengths[g] > 0 ? seq / lengths[g] / G : 0.0;
    s_kl[g] = kls;
    s_clip[g] = ncl;
    s_n[g] = lengths[g];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double pol = 0, k = 0, c = 0, n = 0;
    for (int g = 0; g < G; ++g) {
      pol += s_pol[g];
      k += s_kl[g];
      c += s_clip[g];
      n += s_n[g];
    }
    const double mean_kl = n > 0 ? k / n : 0.0;
    out[0] = pol - beta * mean_kl;
    out[1] = mean_kl;
    out[2] = n > 0 ? c / n : 0.0;
    out[3] = n;
  }
}

}  // namespace

void grpo_stats(const float* lp, const float* old_lp, const float* lp_ref, const float* kl,
                const float* adv, const int* lengths, int G, double clip_eps, double kl_beta,
                int sampled_kl, double* out4, cudaStream_t s) {
  MRSP_REQUIRE(G >= 1 && G <= 1024, MRSP_INVALID_ARGUMENT, "grpo_stats: 1 <= G <= 1024");
  MRSP_REQUIRE(sampled_kl ? lp_ref != nullptr : kl != nullptr, MRSP_INVALID_ARGUMENT,
               "grpo_stats: missing KL input");
  grpo_stats_kernel<<<1, 128, 0, s>>>(lp, old_lp, lp_ref, kl, adv, lengths, G, clip_eps, kl_beta,
                                      sampled_kl, out4);
  count_launch();
  MRSP_CUDA(cudaGetLastError());
}

}  // namespace mrsp

extern "C" mrsp_status mrsp_op_grpo_stats(const float* logprob, const float* old_logprob,
                                          const float* ref_logprob, const float* kl,
                                          const float* advantages, const int32_t* lengths, int G,
                                          double clip_eps, double kl_beta, int sampled_kl,
                                          double* out4, void* stream) {
  return mrsp::guard([&] {
    mrsp::require_device();
    mrsp::grpo_stats(logprob, old_logprob, ref_logprob, kl, advantages, lengths, G, clip_eps,
                     kl_beta, sampled_kl, out4, static_cast<cudaStream_t>(stream));
  });
}
