"""CPU: the float64 autograd GRPO objective (oracle/transformer_grad.py) is
pinned to the reference's analytic gradient and to the forward twin.

* dJ/dlogits from autograd equals grpo_gradient's per-position g
  (/root/reference/proj/src/grpo.cpp:122-206): coeff (onehot(y) - pi) with
  coeff = tok_w A ratio off the clip plateau, plus kl_w pi (lp - lq - KL)
  (exact KL) or kl_w (1 - e^(lq_y - lp_y)) (onehot - pi) (k3), kl_w = -beta/n.
* The policy log-probs of its forward equal oracle/transformer_torch.py's
  (itself pinned to the numpy oracle and HF transformers) at c1.
"""
import numpy as np
import pytest
import torch

from oracle import transformer as T
from oracle import transformer_grad as TG
from oracle import transformer_torch as TT


def analytic_g(lp_all, lq_all, tg, old, adv, lengths, eps, beta, sampled):
    """grpo.cpp:122-206 restated per position (numpy float64)."""
    lp_all, lq_all = lp_all.numpy(), lq_all.numpy()
    n, V = lp_all.shape
    G = len(lengths)
    out = np.zeros_like(lp_all)
    kl_w = -beta / n
    t = 0
    for i in range(G):
        tok_w = 1.0 / (G * lengths[i])
        for _ in range(lengths[i]):
            y = int(tg[t])
            lp, lq = lp_all[t], lq_all[t]
            pi = np.exp(lp)
            ratio = np.exp(lp[y] - old[t])
            plateau = (adv[i] > 0 and ratio > 1 + eps) or (adv[i] < 0 and ratio < 1 - eps)
            g = np.zeros(V)
            if adv[i] != 0 and not plateau:
                coeff = tok_w * adv[i] * ratio
                g -= coeff * pi
                g[y] += coeff
            if beta != 0:
                if sampled:
                    coeff = kl_w * (1.0 - np.exp(lq[y] - lp[y]))
                    g -= coeff * pi
                    g[y] += coeff
                else:
                    kl = float((pi * (lp - lq)).sum())
                    g += kl_w * pi * (lp - lq - kl)
            out[t] = g
            t += 1
    return out


@pytest.mark.parametrize("sampled", [False, True])
def test_autograd_objective_matches_reference_gradient(sampled):
    rng = np.random.default_rng(7)
    lengths = np.array([3, 5, 1, 4])
    n, V = int(lengths.sum()), 11
    logits = torch.tensor(rng.normal(size=(n, V)) * 2, dtype=torch.float64, requires_grad=True)
    ref = torch.tensor(rng.normal(size=(n, V)) * 2, dtype=torch.float64)
    tg = torch.tensor(rng.integers(0, V, n))
    lp_all = torch.log_softmax(logits, -1)
    lq_all = torch.log_softmax(ref, -1)
    lp_y = lp_all.detach().gather(1, tg[:, None])[:, 0].numpy()
    # ratios well inside and well outside the clip window
    old = lp_y - rng.choice([-0.5, -0.05, 0.05, 0.5], size=n)
    adv = np.array([1.0, -0.7, 0.0, 0.4])
    J, stats, _ = TG.objective(lp_all, lq_all, tg, old, adv, lengths, 0.2, 0.05, sampled)
    J.backward()
    want = analytic_g(lp_all.detach(), lq_all, tg, old, adv, lengths, 0.2, 0.05, sampled)
    np.testing.assert_allclose(logits.grad.numpy(), want, rtol=1e-10, atol=1e-14)
    assert stats["token_count"] == n


def test_forward_matches_twin_c1():
    from paper_2507_07966_b200 import engine as E
    w = E.workloads()["c1"]
    c = T.Cfg.from_any(w.cfg)
    grp = E.make_group(w, seed=3)
    emb = torch.tensor(np.random.default_rng(1).normal(size=(w.frames * c.T, c.dim)) * 0.5)
    emb = TT._b(emb)
    want, _ = TT.llm_logprobs(c, 3, "policy.", emb, grp.question, grp.resp, grp.lengths, "cpu")
    P = TG.llm_params(c, 3, "policy.", "cpu", grad=False)
    xs, tg = TG.final_hidden(c, P, emb, grp.question, grp.resp, grp.lengths, "cpu")
    lp = torch.log_softmax(xs @ P["lm_head.weight"].T, -1).gather(1, tg[:, None])[:, 0]
    np.testing.assert_allclose(lp.numpy(), want, rtol=0, atol=1e-9)
