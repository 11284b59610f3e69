"""GPU: the backward of the toy policy on the device (
csrc/toy.cu toy_backward, mrsp_toy_grpo_gradient / mrsp_toy_sft_loss_and_grad)
against the reference's own analytic gradients (golden fixture "backward") and
the CPU oracle (itself bit-exact to the reference, tests/test_backward_oracle.py).

Tolerance: the device evaluates the reference's operations in its order with
explicit rounding and glibc's tanh, but CUDA's fp64 exp / log (<= 1 ulp from
glibc's), so gradients agree to rtol 1e-10 / atol 1e-13 and the scalar stats to
1e-12; token counts and clip fractions exactly. Every SP degree gives the same
bits (the parameter sums run in the serial position order)."""
import json
import pathlib

import numpy as np
import pytest

from oracle import toy
from paper_2507_07966_b200 import mrsp
from paper_2507_07966_b200._lib import InvalidArgument

import test_backward_oracle as O

pytestmark = pytest.mark.gpu
RTOL, ATOL = 1e-10, 1e-13


def params(theta, V, d, h):
    return mrsp.PolicyParams(V, d, h, np.asarray(theta, dtype=np.float64))


def group_of(toks, olds, adv):
    return mrsp.RolloutGroup([mrsp.Rollout(t, o) for t, o in zip(toks, olds)], list(adv))


def close_stats(got, want):
    assert got.token_count == want["token_count"]
    assert got.clip_fraction == want["clip_fraction"]
    assert abs(got.objective - want["objective"]) <= 1e-12
    assert abs(got.mean_kl - want["mean_kl"]) <= 1e-12


@pytest.mark.parametrize("variant,cfg", [
    ("exact_kl", mrsp.GrpoConfig()),
    ("sampled_kl", mrsp.GrpoConfig(sampled_kl=True)),
    ("no_kl", mrsp.GrpoConfig(kl_beta=0.0))])
@pytest.mark.parametrize("sp", [1, 2, 3, 4])
def test_grpo_gradient_vs_reference_golden(gpu, variant, cfg, sp):
    bw, toks, olds, adv = O.golden_case()
    th, rf = params(bw["theta"], O.V, O.D, O.H), params(bw["ref"], O.V, O.D, O.H)
    seq = mrsp.MultimodalSequence(np.array(bw["frame_embeddings"]), bw["text_tokens"])
    grad, st = mrsp.grpo_gradient(group_of(toks, olds, adv), th, rf, seq, cfg, sp_degree=sp)
    np.testing.assert_allclose(grad, bw["grad_" + variant], rtol=RTOL, atol=ATOL)
    close_stats(st, bw["stats_" + variant])


def test_sp_degrees_bit_identical(gpu):
    bw, toks, olds, adv = O.golden_case()
    th, rf = params(bw["theta"], O.V, O.D, O.H), params(bw["ref"], O.V, O.D, O.H)
    seq = mrsp.MultimodalSequence(np.array(bw["frame_embeddings"]), bw["text_tokens"])
    g = group_of(toks, olds, adv)
    base, st0 = mrsp.grpo_gradient(g, th, rf, seq, mrsp.GrpoConfig(), sp_degree=1)
    for sp in (2, 3, 4, 8, 13):  # 13 > longest rollout: idle ranks
        got, st = mrsp.grpo_gradient(g, th, rf, seq, mrsp.GrpoConfig(), sp_degree=sp)
        assert np.array_equal(got, base) and st == st0, sp


@pytest.mark.parametrize("sp", [1, 3])
def test_sft_vs_reference_golden(gpu, sp):
    bw, *_ = O.golden_case()
    th = params(bw["theta"], O.V, O.D, O.H)
    seq = mrsp.MultimodalSequence(np.array(bw["frame_embeddings"]), bw["text_tokens"])
    loss, grad = mrsp.sft_loss_and_grad(th, seq, bw["sft_target"], sp_degree=sp)
    assert abs(loss - bw["sft_loss"]) <= 1e-12
    np.testing.assert_allclose(grad, bw["sft_grad"], rtol=RTOL, atol=ATOL)


CASES = [  # (V, d, h, G, max_len): shapes incl. degenerate dims and long rollouts
    (12, 5, 7, 4, 6), (2, 1, 1, 2, 3), (40, 16, 32, 8, 12), (7, 3, 2, 1, 1), (32, 8, 12, 3, 64)]


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("sampled,beta", [(False, 0.04), (True, 0.04), (False, 0.0), (True, 0.0)])
def test_grpo_gradient_vs_oracle(gpu, case, sampled, beta):
    V, d, h, G, L = case
    for seed in range(3):
        theta, ref, fe, text, toks, olds, adv, _ = O.random_case(seed, V, d, h, G, L)
        want, wst = toy.grpo_gradient(theta, ref, V, d, h, fe, text, toks, olds, adv,
                                      kl_beta=beta, sampled_kl=sampled)
        seq = mrsp.MultimodalSequence(fe, text)
        cfg = mrsp.GrpoConfig(kl_beta=beta, sampled_kl=sampled)
        got, st = mrsp.grpo_gradient(group_of(toks, olds, adv), params(theta, V, d, h),
                                     params(ref, V, d, h), seq, cfg, sp_degree=1 + seed)
        np.testing.assert_allclose(got, want, rtol=RTOL, atol=ATOL)
        close_stats(st, wst)


def test_degenerate_group_has_only_the_kl_gradient(gpu):
    # compute_advantages returns all zeros for a degenerate group (grpo.hpp:29-31):
    # no policy term, the gradient is the KL penalty's alone; with kl_beta = 0 it is 0
    theta, ref, fe, text, toks, olds, _, (V, d, h) = O.random_case(5)
    adv = np.zeros(len(toks))
    seq = mrsp.MultimodalSequence(fe, text)
    g = group_of(toks, olds, adv)
    got, st = mrsp.grpo_gradient(g, params(theta, V, d, h), params(ref, V, d, h), seq,
                                 mrsp.GrpoConfig(kl_beta=0.0))
    assert not got.any() and st.objective == 0.0 and st.clip_fraction == 0.0
    got, _ = mrsp.grpo_gradient(g, params(theta, V, d, h), params(ref, V, d, h), seq,
                                mrsp.GrpoConfig())
    want, _ = toy.grpo_gradient(theta, ref, V, d, h, fe, text, toks, olds, adv)
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=ATOL)


def test_theta_equals_ref_ratio_one(gpu):
    # acceptance criterion 3 shape: theta = ref and old = current log-probs ->
    # ratio 1, KL 0, objective = mean advantage-weighted 1
    theta, _, fe, text, toks, _, adv, (V, d, h) = O.random_case(7)
    ctx = toy.context_vector(theta, V, d, fe, text)
    olds = []
    for t in toks:
        lp, prev = [], 1
        for y in t:
            lp.append(toy.log_softmax(toy.step_logits(theta, V, d, h, ctx, prev))[y])
            prev = y
        olds.append(lp)
    p = params(theta, V, d, h)
    got, st = mrsp.grpo_gradient(group_of(toks, olds, adv), p, p,
                                 mrsp.MultimodalSequence(fe, text), mrsp.GrpoConfig())
    assert abs(st.mean_kl) <= 1e-15 and st.clip_fraction == 0.0
    assert abs(st.objective - np.mean(adv)) <= 1e-12
    want, _ = toy.grpo_gradient(theta, theta, V, d, h, fe, text, toks, olds, adv)
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=ATOL)


def test_errors(gpu):
    theta, ref, fe, text, toks, olds, adv, (V, d, h) = O.random_case(1)
    p, r = params(theta, V, d, h), params(ref, V, d, h)
    seq = mrsp.MultimodalSequence(fe, text)
    cfg = mrsp.GrpoConfig()
    with pytest.raises(InvalidArgument):
        mrsp.grpo_gradient(mrsp.RolloutGroup([], []), p, r, seq, cfg)
    with pytest.raises(InvalidArgument):
        mrsp.grpo_gradient(group_of([[]] + toks[1:], [[]] + olds[1:], adv), p, r, seq, cfg)
    bad = [list(t) for t in toks]
    bad[0][0] = V  # token out of range
    with pytest.raises(InvalidArgument):
        mrsp.grpo_gradient(group_of(bad, olds, adv), p, r, seq, cfg)
    with pytest.raises(InvalidArgument):
        mrsp.grpo_gradient(group_of(toks, olds, adv), p, r,
                           mrsp.MultimodalSequence(np.zeros((0, d)), []), cfg)
    with pytest.raises(InvalidArgument):
        mrsp.sft_loss_and_grad(p, seq, [])
    with pytest.raises(InvalidArgument):
        mrsp.sft_loss_and_grad(p, seq, [0, V])
    one = params(np.zeros(1 * 1 + 2 * 1 + 1 + 1 + 1), 1, 1, 1)  # V = 1: prev = EOS out of range
    with pytest.raises(InvalidArgument):
        mrsp.sft_loss_and_grad(one, mrsp.MultimodalSequence(np.zeros((1, 1)), []), [0])
