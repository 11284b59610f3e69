"""CPU restatement of the GRPO token terms — TEST INFRASTRUCTURE ONLY.

evaluate_from_logits, /root/reference/proj/src/grpo.cpp:68-108, given the
per-token log-probs instead of logits. Pinned against the reference's own
GroupStats in tests/golden/ref_toy.json ("grpo", produced by
oracle/gen_golden.cpp via grpo_objective).
"""
import math


def group_stats(lps, olds, refs, kls, adv, clip_eps, kl_beta, sampled_kl=False):
    G = float(len(lps))
    policy_term, kl_sum, n_tok, n_clip = 0.0, 0.0, 0, 0
    for i in range(len(lps)):
        a = adv[i]
        seq = 0.0
        for t in range(len(lps[i])):
            ratio = math.exp(lps[i][t] - olds[i][t])
            clipped = min(max(ratio, 1.0 - clip_eps), 1.0 + clip_eps)
            seq += min(ratio * a, clipped * a)
            if (a > 0 and ratio > 1.0 + clip_eps) or (a < 0 and ratio < 1.0 - clip_eps):
                n_clip += 1
            if sampled_kl:
                lr = refs[i][t] - lps[i][t]
                kl_sum += math.exp(lr) - 1.0 - lr
            else:
                kl_sum += kls[i][t]
            n_tok += 1
        policy_term += seq / len(lps[i]) / G
    mean_kl = kl_sum / n_tok
    return {"objective": policy_term - kl_beta * mean_kl, "mean_kl": mean_kl,
            "clip_fraction": n_clip / n_tok, "token_count": n_tok}
