"""CPU: the oracle's restatement of the backward (grpo_gradient, grpo.cpp:122-206;
sft_loss_and_grad, grpo.cpp:208-223; GradAccumulator, policy.cpp:195-260) —
pinned bit for bit to the reference's own analytic gradients (golden fixture
"backward", made by oracle/gen_golden.cpp linked against the reference
sources) and checked against central finite differences of the objective, as
the reference's acceptance criterion 1 does (acceptance.cpp:132-210)."""
import json
import pathlib

import numpy as np
import pytest

from oracle import toy

ROOT = pathlib.Path(__file__).resolve().parents[1]
GOLD = json.loads((ROOT / "tests" / "golden" / "ref_toy.json").read_text())
V, D, H = 32, 8, 12


def golden_case():
    bw, g = GOLD["backward"], GOLD["grpo"]
    toks = [r["tokens"] for r in g["rollouts"]]
    olds = [r["old_logprobs"] for r in g["rollouts"]]
    return bw, toks, olds, g["advantages"]


@pytest.mark.parametrize("variant,kw", [("exact_kl", {}), ("sampled_kl", {"sampled_kl": True}),
                                        ("no_kl", {"kl_beta": 0.0})])
def test_grpo_gradient_golden_bit_exact(variant, kw):
    bw, toks, olds, adv = golden_case()
    grad, st = toy.grpo_gradient(bw["theta"], bw["ref"], V, D, H, bw["frame_embeddings"],
                                 bw["text_tokens"], toks, olds, adv, **kw)
    assert grad.tolist() == bw["grad_" + variant]
    assert st == bw["stats_" + variant]


def test_sft_golden_bit_exact():
    bw, *_ = golden_case()
    loss, grad = toy.sft_loss_and_grad(bw["theta"], V, D, H, bw["frame_embeddings"],
                                       bw["text_tokens"], bw["sft_target"])
    assert loss == bw["sft_loss"] and grad.tolist() == bw["sft_grad"]


def random_case(seed, V=12, d=5, h=7, G=4, max_len=6):
    rng = np.random.default_rng(seed)
    theta = toy.policy_random(V, d, h, 100 + seed, 0.5)
    ref = toy.policy_random(V, d, h, 200 + seed, 0.5)
    fe = np.tanh(rng.normal(size=(3, d)))
    text = rng.integers(0, V, size=3)
    toks = [rng.integers(0, V, size=int(rng.integers(1, max_len + 1))).tolist() for _ in range(G)]
    # old log-probs near the current ones so ratios straddle the clip range
    olds = []
    for t in toks:
        ctx = toy.context_vector(theta, V, d, fe, text)
        lp, prev = [], 1
        for y in t:
            lp.append(toy.log_softmax(toy.step_logits(theta, V, d, h, ctx, prev))[y])
            prev = y
        olds.append((np.array(lp) + rng.normal(scale=0.3, size=len(t))).tolist())
    adv = rng.normal(size=G)
    return theta, ref, fe, text, toks, olds, adv, (V, d, h)


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("sampled", [False, True])
def test_grpo_gradient_matches_finite_differences(seed, sampled):
    theta, ref, fe, text, toks, olds, adv, (V_, d, h) = random_case(seed)
    an, _ = toy.grpo_gradient(theta, ref, V_, d, h, fe, text, toks, olds, adv,
                              sampled_kl=sampled)

    def J(th):
        return toy.grpo_gradient(th, ref, V_, d, h, fe, text, toks, olds, adv,
                                 sampled_kl=sampled)[1]["objective"]

    eps = 1e-6
    fd = np.array([(J(theta + eps * e) - J(theta - eps * e)) / (2 * eps)
                   for e in np.eye(theta.shape[0])])
    # the clipped surrogate is piecewise smooth; a probe straddling a clip
    # boundary is the only way FD can disagree, so compare with a norm bound
    err = np.linalg.norm(an - fd) / max(np.linalg.norm(fd), 1e-12)
    assert err < 1e-4, err


@pytest.mark.parametrize("seed", range(3))
def test_sft_gradient_matches_finite_differences(seed):
    theta, _, fe, text, toks, *_ , (V_, d, h) = random_case(seed)
    target = toks[0] + [1]
    _, an = toy.sft_loss_and_grad(theta, V_, d, h, fe, text, target)
    eps = 1e-6
    fd = np.array([(toy.sft_loss_and_grad(theta + eps * e, V_, d, h, fe, text, target)[0] -
                    toy.sft_loss_and_grad(theta - eps * e, V_, d, h, fe, text, target)[0]) / (2 * eps)
                   for e in np.eye(theta.shape[0])])
    assert np.abs(an - fd).max() <= 1e-6 * max(1.0, np.abs(fd).max())
