"""GRPO gradient of the transformer-shaped policy by float64 autograd — TEST
INFRASTRUCTURE (imported only by tests/ and tools/).

The reference differentiates its toy policy analytically: grpo_gradient
(/root/reference/proj/src/grpo.cpp:122-206) forms g = dJ/dlogits per scored
position — the clipped-ratio term (grpo.cpp:152-160, zero on the clip plateau)
and the exact-KL term g += kl_w pi (lp - lq - KL) with kl_w = -beta / tokens
(:170-176) or the sampled k3 term (:162-168) — and GradAccumulator
(policy.cpp:195-260) back-propagates it. This module states the same objective

    J = sum_g sum_t min(r A_g, clip(r, 1 - eps, 1 + eps) A_g) / len_g / G
        - beta * mean_t KL_t,          r = exp(lp_t - old_t)

(evaluate_from_logits, grpo.cpp:68-108) on top of the transformer-shaped
forward of oracle/transformer_torch.py (same counter-based weights, same bf16 /
fp32 storage roundings, same MR-SP packed layout and mask, teacher forcing with
EOS at t = 0), with every policy-LLM tensor a float64 leaf, and lets torch
autograd produce dJ/dtheta. Roundings are differentiated as the identity (a
cast's gradient), which is what the device backward computes too. The video
embeddings are inputs (the vision tower is frozen, as the reference's policy
parameters exclude its encoder, policy.hpp:39-53).

Dense L x L attention: for the small parity configurations only.
"""
from __future__ import annotations

import math
from typing import Dict

import numpy as np
import torch

from . import transformer as T
from . import transformer_torch as TT

F64 = torch.float64


def _leaf(t: torch.Tensor) -> torch.Tensor:
    return t.detach().clone().requires_grad_(True)


def llm_params(c: T.Cfg, seed: int, prefix: str, dev, grad: bool) -> Dict[str, torch.Tensor]:
    """All LLM tensors under the HF names the engine's save_grads uses."""
    d, hd, nq, nkv = c.dim, c.head_dim, c.n_q_heads, c.n_kv_heads
    P = {"model.embed_tokens.weight": TT.init_bf16((c.vocab, d), seed, prefix + "embed", T.K_EMBED, dev),
         "model.norm.weight": TT.init_f32((d,), seed, prefix + "final_norm", T.K_NORM, 1.0, dev),
         "lm_head.weight": TT.init_bf16((c.vocab, d), seed, prefix + "lm_head", T.wscale(d), dev)}
    for l in range(c.layers):
        W = TT.llm_layer_weights(c, seed, prefix, l, dev)
        p = f"model.layers.{l}."
        P[p + "input_layernorm.weight"] = W["attn_norm"]
        P[p + "self_attn.q_proj.weight"] = W["wqkv"][:nq * hd]
        P[p + "self_attn.k_proj.weight"] = W["wqkv"][nq * hd:(nq + nkv) * hd]
        P[p + "self_attn.v_proj.weight"] = W["wqkv"][(nq + nkv) * hd:]
        P[p + "self_attn.q_proj.bias"] = W["bqkv"][:nq * hd]
        P[p + "self_attn.k_proj.bias"] = W["bqkv"][nq * hd:(nq + nkv) * hd]
        P[p + "self_attn.v_proj.bias"] = W["bqkv"][(nq + nkv) * hd:]
        P[p + "self_attn.o_proj.weight"] = W["wo"]
        P[p + "post_attention_layernorm.weight"] = W["mlp_norm"]
        P[p + "mlp.gate_proj.weight"] = W["w_gate"]
        P[p + "mlp.up_proj.weight"] = W["w_up"]
        P[p + "mlp.down_proj.weight"] = W["w_down"]
    return {k: (_leaf(v) if grad else v.detach()) for k, v in P.items()}


def _b(x: torch.Tensor) -> torch.Tensor:
    """bf16 storage rounding (TT._b) with a float64 straight-through gradient
    (a plain cast would round the gradient to bf16 as well)."""
    return x + (TT._b(x.detach()) - x.detach())


def _s(x: torch.Tensor) -> torch.Tensor:
    return x + (TT._s(x.detach()) - x.detach())


def _rms(x, w, eps):
    r = 1.0 / torch.sqrt((x * x).mean(-1, keepdim=True) + eps)
    return _b(w * (x * r))


def _rope(x, cos, sin):
    x1, x2 = x[..., :64], x[..., 64:]
    cc, ss = cos[:, None, :], sin[:, None, :]
    return _b(torch.cat([x1 * cc - x2 * ss, x2 * cc + x1 * ss], -1))


class _AttnBf16Bwd(torch.autograd.Function):
    """MR-SP attention whose backward rounds what the device rounds: dO, the
    stored O, P and dS to bf16 (the tcgen05 operands), D = rowsum(dO o O) from
    the bf16 values (csrc/backward.cu). Forward: exact float64 softmax."""

    @staticmethod
    def forward(ctx, q, k, v, mask, scale):  # q [L, nq, hd], k / v [L, nq, hd] (repeated)
        s = torch.einsum("qhd,khd->hqk", q, k) * scale
        s = s.masked_fill(~mask[None], float("-inf"))
        p = torch.softmax(s, -1)
        o = torch.einsum("hqk,khd->qhd", p, v)
        ctx.save_for_backward(q, k, v, p, o)
        ctx.scale = scale
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, p, o = ctx.saved_tensors
        bf = lambda x: TT._b(x)
        do_b, o_b = bf(do), bf(o)
        dp = torch.einsum("qhd,khd->hqk", do_b, v)
        D = (do_b * o_b).sum(-1).t()[:, :, None]  # [h, q, 1]
        ds = bf(p * (dp - D))
        dq = torch.einsum("hqk,khd->qhd", ds, k) * ctx.scale
        dk = torch.einsum("hqk,qhd->khd", ds, q) * ctx.scale
        dv = torch.einsum("hqk,qhd->khd", bf(p), do_b)
        return dq, dk, dv, None, None


def final_hidden(c: T.Cfg, P, frame_emb: torch.Tensor, question, resp, lengths, dev,
                 emulate_bf16_attn_bwd: bool = False):
    """Final-normed hidden rows at the scored positions (row-major over (g, j))."""
    n_frame_tok = frame_emb.shape[0]
    tok, pos, pad, Lp, L = T.pack(n_frame_tok, question, resp, lengths)
    resp = np.asarray(resp)
    G, Lmax = resp.shape
    d, hd, nq, nkv = c.dim, c.head_dim, c.n_q_heads, c.n_kv_heads
    rep = nq // nkv
    E = P["model.embed_tokens.weight"]
    txt = torch.as_tensor(tok[n_frame_tok:].astype(np.int64), device=dev)
    h = torch.cat([frame_emb.to(dev, F64), E[txt]], 0)
    cos, sin = TT.rope_tables(c, pos, dev)
    mask = torch.as_tensor(T.mrsp_mask(L, Lp, Lmax), device=dev)
    scale = 1.0 / math.sqrt(hd)
    for l in range(c.layers):
        p = f"model.layers.{l}."
        xn = _rms(h, P[p + "input_layernorm.weight"], c.rms_eps)
        wqkv = torch.cat([P[p + "self_attn.q_proj.weight"], P[p + "self_attn.k_proj.weight"],
                          P[p + "self_attn.v_proj.weight"]], 0)
        bqkv = torch.cat([P[p + "self_attn.q_proj.bias"], P[p + "self_attn.k_proj.bias"],
                          P[p + "self_attn.v_proj.bias"]], 0)
        qkv = _b(xn @ wqkv.T + bqkv)
        q = _rope(qkv[:, :nq * hd].reshape(L, nq, hd), cos, sin)
        k = _rope(qkv[:, nq * hd:(nq + nkv) * hd].reshape(L, nkv, hd), cos, sin)
        v = qkv[:, (nq + nkv) * hd:].reshape(L, nkv, hd)
        kk = k.repeat_interleave(rep, 1)  # [L, nq, hd] (head h uses kv head h // rep)
        vv = v.repeat_interleave(rep, 1)
        if emulate_bf16_attn_bwd:
            o = _b(_AttnBf16Bwd.apply(q, kk, vv, mask, scale).reshape(L, nq * hd))
        else:
            s = torch.einsum("qhd,khd->hqk", q, kk) * scale
            s = s.masked_fill(~mask[None], float("-inf"))
            pr = torch.softmax(s, -1)
            o = _b(torch.einsum("hqk,khd->qhd", pr, vv).reshape(L, nq * hd))
        h = _s(h + o @ P[p + "self_attn.o_proj.weight"].T)
        xn = _rms(h, P[p + "post_attention_layernorm.weight"], c.rms_eps)
        g_ = _s(xn @ P[p + "mlp.gate_proj.weight"].T)
        u_ = _s(xn @ P[p + "mlp.up_proj.weight"].T)
        act = _b(TT.silu(g_) * u_)
        h = _s(h + act @ P[p + "mlp.down_proj.weight"].T)
    rows = [Lp + g * Lmax + j for g in range(G) for j in range(int(lengths[g]))]
    tg = [int(resp[g, j]) for g in range(G) for j in range(int(lengths[g]))]
    xs = _rms(h[torch.as_tensor(rows, device=dev)], P["model.norm.weight"], c.rms_eps)
    return xs, torch.as_tensor(tg, device=dev)


def objective(lp_all, lq_all, tg, old_lp, adv, lengths, clip_eps: float, kl_beta: float,
              sampled_kl: bool):
    """J of evaluate_from_logits (grpo.cpp:68-108) from per-token log-softmax rows
    [n, V] of the policy (differentiable) and the reference; returns (J, stats)."""
    dev = lp_all.device
    lp = lp_all.gather(1, tg[:, None])[:, 0]
    lq = lq_all.gather(1, tg[:, None])[:, 0]
    lengths = np.asarray(lengths)
    G, n = len(lengths), int(lengths.sum())
    old = torch.as_tensor(np.asarray(old_lp, dtype=np.float64), device=dev)
    A = torch.as_tensor(np.repeat(np.asarray(adv, dtype=np.float64), lengths), device=dev)
    tok_w = torch.as_tensor(np.repeat(1.0 / (G * lengths.astype(np.float64)), lengths), device=dev)
    ratio = torch.exp(lp - old)
    term = torch.minimum(ratio * A, torch.clamp(ratio, 1.0 - clip_eps, 1.0 + clip_eps) * A)
    policy = (term * tok_w).sum()
    if sampled_kl:
        lr = lq - lp
        kl_t = torch.exp(lr) - 1.0 - lr
    else:
        kl_t = (torch.exp(lp_all) * (lp_all - lq_all)).sum(-1)
    mean_kl = kl_t.sum() / n
    J = policy - kl_beta * mean_kl
    with torch.no_grad():
        clipped = ((A > 0) & (ratio > 1 + clip_eps)) | ((A < 0) & (ratio < 1 - clip_eps))
    stats = {"objective": float(J.detach()), "mean_kl": float(mean_kl.detach()),
             "clip_fraction": float(clipped.double().mean()), "token_count": float(n)}
    return J, stats, lp


def grpo_objective_grad(c: T.Cfg, policy_seed: int, ref_seed: int, frame_emb, question, resp,
                        lengths, old_lp, adv, clip_eps: float, kl_beta: float, sampled_kl: bool,
                        dev="cpu", emulate_bf16_attn_bwd: bool = False):
    """(stats, policy log-probs, {HF name: dJ/dtheta as float64 numpy}).
    emulate_bf16_attn_bwd: the attention backward rounds dO, O, P and dS to bf16
    as the device does (the dominant rounding of the q / k gradients); the
    default is the exact float64 gradient."""
    c = T.Cfg.from_any(c)
    P = llm_params(c, policy_seed, "policy.", dev, grad=True)
    R = llm_params(c, ref_seed, "ref.", dev, grad=False)
    xs, tg = final_hidden(c, P, frame_emb, question, resp, lengths, dev, emulate_bf16_attn_bwd)
    with torch.no_grad():
        xr, _ = final_hidden(c, R, frame_emb, question, resp, lengths, dev)
    lp_all = torch.log_softmax(xs @ P["lm_head.weight"].T, -1)
    lq_all = torch.log_softmax(xr @ R["lm_head.weight"].T, -1)
    J, stats, lp = objective(lp_all, lq_all, tg, old_lp, adv, lengths, clip_eps, kl_beta,
                             sampled_kl)
    J.backward()
    grads = {k: v.grad.detach().cpu().numpy() for k, v in P.items()}
    return stats, lp.detach().cpu().numpy(), grads


def sft_loss_grad(c: T.Cfg, policy_seed: int, frame_emb, question, resp, lengths, dev="cpu",
                  emulate_bf16_attn_bwd: bool = False):
    """sft_loss_and_grad (grpo.cpp:208-223) over the G teacher-forced rows:
    loss = mean over all row tokens of -log pi(y); (loss, log-probs, grads of the loss)."""
    c = T.Cfg.from_any(c)
    P = llm_params(c, policy_seed, "policy.", dev, grad=True)
    xs, tg = final_hidden(c, P, frame_emb, question, resp, lengths, dev, emulate_bf16_attn_bwd)
    lp = torch.log_softmax(xs @ P["lm_head.weight"].T, -1).gather(1, tg[:, None])[:, 0]
    loss = -lp.mean()
    loss.backward()
    grads = {k: v.grad.detach().cpu().numpy() for k, v in P.items()}
    return float(loss.detach()), lp.detach().cpu().numpy(), grads
