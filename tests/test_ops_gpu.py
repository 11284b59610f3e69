"""GPU: HBM-bound device operators and the fused LM-head log-prob vs plain
PyTorch fp32 references (through the C-ABI)."""
import ctypes
import math

import numpy as np
import pytest
import torch

from oracle import transformer as T
from paper_2507_07966_b200 import _lib

pytestmark = pytest.mark.gpu


def vp(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


@pytest.mark.parametrize("M,V,K", [(77, 32, 256), (300, 152064, 512), (1030, 5000, 3584)])
def test_lmhead_logprob(gpu, M, V, K):
    g = torch.Generator(device="cuda").manual_seed(M + V)
    X = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    W = (torch.randn(V, K, device="cuda", generator=g) / K ** 0.5 * 3).bfloat16()
    tgt = torch.randint(0, V, (M,), device="cuda", dtype=torch.int32, generator=g)
    lp = torch.empty(M, device="cuda")
    lse = torch.empty(M, device="cuda")
    wsb = _lib.lib().mrsp_lmhead_workspace_bytes(M, V)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    _lib.check(_lib.lib().mrsp_op_lmhead_logprob(vp(X), K, vp(W), M, V, K, vp(tgt), vp(lp), vp(lse),
                                                 vp(ws), wsb, None))
    logits = X.double() @ W.double().T
    want = torch.log_softmax(logits, -1).gather(1, tgt.long()[:, None])[:, 0]
    torch.cuda.synchronize()
    assert (lp.double() - want).abs().max().item() < 2e-3
    assert (lse.double() - torch.logsumexp(logits, -1)).abs().max().item() < 2e-3


def test_rmsnorm_and_gather(gpu):
    n, d = 333, 3584
    x = torch.randn(n, d, device="cuda") * 3
    w = 1 + 0.1 * torch.randn(d, device="cuda")
    out = torch.empty(n, d, device="cuda", dtype=torch.bfloat16)
    _lib.check(_lib.lib().mrsp_op_rmsnorm(vp(x), d, vp(w), vp(out), d, n, d, 1e-6, None, None))
    want = w * (x * torch.rsqrt((x * x).mean(-1, keepdim=True) + 1e-6))
    assert ((out.float() - want).abs() / (want.abs() + 1e-2)).max().item() < 1e-2
    rows = torch.tensor([5, 0, 332, 17], device="cuda", dtype=torch.int32)
    out2 = torch.empty(4, d, device="cuda", dtype=torch.bfloat16)
    _lib.check(_lib.lib().mrsp_op_rmsnorm(vp(x), d, vp(w), vp(out2), d, 4, d, 1e-6, vp(rows), None))
    assert torch.equal(out2, out[rows.long()])


def test_layernorm(gpu):
    n, d = 257, 1152
    x = torch.randn(n, d, device="cuda") * 2 + 0.5
    w = 1 + 0.1 * torch.randn(d, device="cuda")
    b = 0.1 * torch.randn(d, device="cuda")
    out = torch.empty(n, d, device="cuda", dtype=torch.bfloat16)
    _lib.check(_lib.lib().mrsp_op_layernorm(vp(x), d, vp(w), vp(b), vp(out), d, n, d, 1e-6, None))
    want = torch.nn.functional.layer_norm(x, (d,), w, b, 1e-6)
    assert (out.float() - want).abs().max().item() < 3e-2


def test_rope_matches_oracle(gpu):
    n, H = 300, 6
    x = torch.randn(n, H * 128, device="cuda").bfloat16()
    pos = torch.randint(0, 262144, (n,), device="cuda", dtype=torch.int32)
    y = x.clone()
    _lib.check(_lib.lib().mrsp_op_rope(vp(y), H * 128, 0, H, vp(pos), n, 1e6, None))
    c = T.Cfg(64, 8, 8, 1, 8, 8, 1, 8, 1, 1, 128, 128, 1, 8)
    cos, sin = T.rope_tables(c, pos.cpu().numpy())
    want = T.apply_rope(x.float().cpu().numpy().reshape(n, H, 128), cos, sin).reshape(n, H * 128)
    got = y.float().cpu().numpy()
    assert np.abs(got - want).max() <= 2 ** -6 * np.abs(want).max()
    assert (got == want).mean() > 0.97


@pytest.mark.parametrize("F,S,P,kpad", [(3, 224, 14, 592), (5, 64, 8, 192), (2, 30, 6, 112)])
def test_patchify_matches_oracle(gpu, F, S, P, kpad):
    # SigLIP (224^2, patch 14, K padded 588 -> 592), c1 (64^2, patch 8), and a
    # width that is not a multiple of 4 (scalar staging path)
    pix = torch.rand(F, 3 * S * S, device="cuda") * 2 - 1
    out = torch.empty(F * (S // P) ** 2, kpad, device="cuda", dtype=torch.bfloat16)
    _lib.check(_lib.lib().mrsp_op_patchify(vp(pix), vp(out), F, S, S, P, kpad, None))
    want = T.patchify(pix.cpu().numpy(), S, P)
    got = out.float().cpu().numpy()
    kreal = 3 * P * P
    assert np.array_equal(got[:, :kreal], want) and (got[:, kreal:] == 0).all()


@pytest.mark.parametrize("M,V,K", [(77, 32, 256), (300, 152064, 3584), (1000, 5000, 512)])
def test_lmhead_dual_logprob_kl(gpu, M, V, K):
    """Fused policy+reference LM head vs torch fp64: both log-probs and the exact
    KL(p||q) = sum_v p (log p - log q) (grpo.cpp:94-96)."""
    g = torch.Generator(device="cuda").manual_seed(M * 3 + V)
    Xp = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    Xr = (Xp.float() + 0.3 * torch.randn(M, K, device="cuda", generator=g)).bfloat16()
    Wp = (torch.randn(V, K, device="cuda", generator=g) / K ** 0.5 * 2).bfloat16()
    Wr = (Wp.float() + 0.2 * torch.randn(V, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    tgt = torch.randint(0, V, (M,), device="cuda", dtype=torch.int32, generator=g)
    lp_p, lp_r, kl = (torch.empty(M, device="cuda") for _ in range(3))
    wsb = _lib.lib().mrsp_lmhead_dual_workspace_bytes(M, V)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    _lib.check(_lib.lib().mrsp_op_lmhead_dual(vp(Xp), vp(Wp), vp(Xr), vp(Wr), M, V, K, vp(tgt),
                                              vp(lp_p), vp(lp_r), vp(kl), vp(ws), wsb, None))
    a = torch.log_softmax(Xp.double() @ Wp.double().T, -1)
    b = torch.log_softmax(Xr.double() @ Wr.double().T, -1)
    want_kl = (a.exp() * (a - b)).sum(-1)
    torch.cuda.synchronize()
    assert (lp_p.double() - a.gather(1, tgt.long()[:, None])[:, 0]).abs().max().item() < 2e-3
    assert (lp_r.double() - b.gather(1, tgt.long()[:, None])[:, 0]).abs().max().item() < 2e-3
    assert (kl.double() - want_kl).abs().max().item() < 2e-3 + 1e-3 * want_kl.abs().max().item()
    assert (kl >= -1e-4).all()


def test_grpo_stats_vs_reference(gpu):
    """Device GRPO token terms vs the reference's own GroupStats (golden)."""
    import json
    import pathlib
    gold = json.loads((pathlib.Path(__file__).parent / "golden" / "ref_toy.json").read_text())["grpo"]
    r = gold["rollouts"]
    cat = lambda k: torch.tensor([v for x in r for v in x[k]], dtype=torch.float32, device="cuda")
    lp, old, ref, kl = cat("logprobs"), cat("old_logprobs"), cat("ref_logprobs"), cat("kl")
    adv = torch.tensor(gold["advantages"], dtype=torch.float32, device="cuda")
    lens = torch.tensor([len(x["tokens"]) for x in r], dtype=torch.int32, device="cuda")
    for key, sampled in (("stats_exact_kl", 0), ("stats_sampled_kl", 1)):
        out = torch.zeros(4, dtype=torch.float64, device="cuda")
        _lib.check(_lib.lib().mrsp_op_grpo_stats(vp(lp), vp(old), vp(ref), vp(kl), vp(adv), vp(lens),
                                                 len(r), gold["clip_eps"], gold["kl_beta"], sampled,
                                                 vp(out), None))
        o = out.cpu().tolist()
        want = gold[key]
        assert o[3] == want["token_count"] and abs(o[2] - want["clip_fraction"]) < 1e-12
        assert abs(o[0] - want["objective"]) < 1e-5 and abs(o[1] - want["mean_kl"]) < 1e-5
