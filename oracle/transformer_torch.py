"""Torch float64 twin of oracle/transformer.py — TEST INFRASTRUCTURE.

Imported only by tests/ and tools/; never by the product package, never by
bench.py's timed leg.

The numpy oracle (oracle/transformer.py, pinned to HF transformers' SigLIP /
Qwen2 in tests/test_oracle_hf_pin.py) is exact but single-threaded numpy with a
dense L x L mask: it finishes c1 and one production-width layer in seconds and
nothing larger. This module restates the SAME algorithm — same counter-based
weights, same storage-rounding boundaries (bf16 activations, fp32 residual,
float32 -> bf16 double rounding exactly as `_b`), same mask, same
teacher-forcing layout, float64 arithmetic — with torch tensors on any device,
so the benchmarked configurations c2..c5 can be checked end to end on the GPU
box in minutes:

  * weights are generated per layer on the device from the same splitmix64
    counters (`init_bf16`/`init_f32`; embedding rows only for the token ids
    used), so a 7.6B-parameter model never sits in memory in float64;
  * vision runs frame chunk by frame chunk (its attention is intra-frame);
  * LLM attention runs per (query block, kv head) over the keys the block can
    see, float64 scores, the MR-SP mask of `mrsp_mask`;
  * the SwiGLU MLP runs in row chunks; the LM head in vocabulary chunks with an
    exact two-pass log-sum-exp (max first, then the shifted sum, as numpy).

Pinned to the numpy oracle in tests/test_oracle_twin.py (CPU): weights
bit-identical, embeddings and log-probs equal to <= 1e-12 relative at c1 and at
production widths. Only matmul summation order differs.
"""
from __future__ import annotations

import math
from typing import Dict, Optional

import numpy as np
import torch

from . import transformer as T

F64 = torch.float64


def _u64(c: int) -> int:
    """uint64 constant as the int64 with the same bits."""
    c &= 0xFFFFFFFFFFFFFFFF
    return c - (1 << 64) if c >= (1 << 63) else c


_G, _M1, _M2 = _u64(0x9E3779B97F4A7C15), _u64(0xBF58476D1CE4E5B9), _u64(0x94D049BB133111EB)


def _shr(z: torch.Tensor, s: int) -> torch.Tensor:
    """Logical right shift of int64 bit patterns."""
    return (z >> s) & ((1 << (64 - s)) - 1)


def splitmix(z: torch.Tensor) -> torch.Tensor:
    """splitmix64 on int64 tensors (two's-complement wrap == uint64 arithmetic)."""
    z = z + _G
    z = (z ^ _shr(z, 30)) * _M1
    z = (z ^ _shr(z, 27)) * _M2
    return z ^ _shr(z, 31)


def _uniform(idx: torch.Tensor, key: int) -> torch.Tensor:
    """2u - 1 in float32 for counters idx (T._uniform_t restated)."""
    u = _shr(splitmix(idx + _u64(key)), 40).to(torch.float32) * (2.0 ** -24)
    return u * 2.0 - 1.0


def _idx(shape, rows, dev) -> torch.Tensor:
    if rows is None:
        return torch.arange(int(np.prod(shape)), dtype=torch.int64, device=dev).reshape(shape)
    rows = torch.as_tensor(rows, dtype=torch.int64, device=dev)
    return rows[:, None] * shape[1] + torch.arange(shape[1], dtype=torch.int64, device=dev)[None]


def init_bf16(shape, seed, name, a, dev, rows=None) -> torch.Tensor:
    """T.init_bf16 as float64 on `dev`; `rows` = only those rows of a 2-D tensor."""
    t = torch.tensor(np.float32(a), device=dev) * _uniform(_idx(shape, rows, dev),
                                                           T.tensor_key(seed, name))
    return t.to(torch.bfloat16).to(F64)


def init_f32(shape, seed, name, a, offset, dev) -> torch.Tensor:
    t = torch.tensor(np.float32(a), device=dev) * _uniform(_idx(shape, None, dev),
                                                           T.tensor_key(seed, name))
    return (t + np.float32(offset)).to(torch.float32).to(F64)


# ------------------------------------------------------------ storage rounding
def _b(x: torch.Tensor) -> torch.Tensor:
    """bf16 storage: float64 -> float32 -> bf16 (both RNE), as T._b."""
    return x.to(torch.float32).to(torch.bfloat16).to(F64)


def _s(x: torch.Tensor) -> torch.Tensor:
    return x.to(torch.float32).to(F64)


def layernorm(x, w, b, eps):
    mu = x.mean(-1, keepdim=True)
    var = ((x - mu) ** 2).mean(-1, keepdim=True)
    return _b((x - mu) / torch.sqrt(var + eps) * w + b)


def rmsnorm(x, w, eps):
    r = 1.0 / torch.sqrt((x * x).mean(-1, keepdim=True) + eps)
    return _b(w * (x * r))


def gelu_tanh(x):
    return 0.5 * x * (1.0 + torch.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))


def silu(x):
    return x / (1.0 + torch.exp(-x))


def linear(x, w, b=None):
    y = x @ w.T
    return y if b is None else y + b


# -------------------------------------------------------------------- weights
def vision_weights(c: T.Cfg, seed: int, dev) -> Dict[str, torch.Tensor]:
    kreal, vd = 3 * c.patch * c.patch, c.v_dim
    ws = T.wscale
    W = {
        "patch_w": init_bf16((vd, kreal), seed, "vision.patch_w", ws(kreal), dev),
        "patch_b": init_f32((vd,), seed, "vision.patch_b", T.K_BIAS, 0.0, dev),
        "pos": init_f32((c.T, vd), seed, "vision.pos", T.K_POS, 0.0, dev),
        "post_w": init_f32((vd,), seed, "vision.post_w", T.K_NORM, 1.0, dev),
        "post_b": init_f32((vd,), seed, "vision.post_b", T.K_BIAS, 0.0, dev),
        "p1_w": init_bf16((c.dim, vd), seed, "proj.w1", ws(vd), dev),
        "p1_b": init_f32((c.dim,), seed, "proj.b1", T.K_BIAS, 0.0, dev),
        "p2_w": init_bf16((c.dim, c.dim), seed, "proj.w2", ws(c.dim), dev),
        "p2_b": init_f32((c.dim,), seed, "proj.b2", T.K_BIAS, 0.0, dev),
    }
    for l in range(c.v_layers):
        p = f"vision.{l}."
        W[p + "ln1_w"] = init_f32((vd,), seed, p + "ln1_w", T.K_NORM, 1.0, dev)
        W[p + "ln1_b"] = init_f32((vd,), seed, p + "ln1_b", T.K_BIAS, 0.0, dev)
        W[p + "wqkv"] = init_bf16((3 * vd, vd), seed, p + "wqkv", ws(vd), dev)
        W[p + "bqkv"] = init_f32((3 * vd,), seed, p + "bqkv", T.K_BIAS, 0.0, dev)
        W[p + "wo"] = init_bf16((vd, vd), seed, p + "wo", ws(vd), dev)
        W[p + "bo"] = init_f32((vd,), seed, p + "bo", T.K_BIAS, 0.0, dev)
        W[p + "ln2_w"] = init_f32((vd,), seed, p + "ln2_w", T.K_NORM, 1.0, dev)
        W[p + "ln2_b"] = init_f32((vd,), seed, p + "ln2_b", T.K_BIAS, 0.0, dev)
        W[p + "w1"] = init_bf16((c.v_mlp, vd), seed, p + "w1", ws(vd), dev)
        W[p + "b1"] = init_f32((c.v_mlp,), seed, p + "b1", T.K_BIAS, 0.0, dev)
        W[p + "w2"] = init_bf16((vd, c.v_mlp), seed, p + "w2", ws(c.v_mlp), dev)
        W[p + "b2"] = init_f32((vd,), seed, p + "b2", T.K_BIAS, 0.0, dev)
    return W


def llm_layer_weights(c: T.Cfg, seed: int, prefix: str, l: int, dev) -> Dict[str, torch.Tensor]:
    """One decoder layer of T.llm_weights (same names and counters)."""
    d, hd = c.dim, c.head_dim
    qkv_rows = (c.n_q_heads + 2 * c.n_kv_heads) * hd
    p, ws = f"{prefix}{l}.", T.wscale
    return {
        "attn_norm": init_f32((d,), seed, p + "attn_norm", T.K_NORM, 1.0, dev),
        "wqkv": init_bf16((qkv_rows, d), seed, p + "wqkv", ws(d), dev),
        "bqkv": init_f32((qkv_rows,), seed, p + "bqkv", T.K_BIAS, 0.0, dev),
        "wo": init_bf16((d, c.n_q_heads * hd), seed, p + "wo", ws(c.n_q_heads * hd), dev),
        "mlp_norm": init_f32((d,), seed, p + "mlp_norm", T.K_NORM, 1.0, dev),
        "w_gate": init_bf16((c.mlp, d), seed, p + "w_gate", ws(d), dev),
        "w_up": init_bf16((c.mlp, d), seed, p + "w_up", ws(d), dev),
        "w_down": init_bf16((d, c.mlp), seed, p + "w_down", ws(c.mlp), dev),
    }


# -------------------------------------------------------------------- stage 1
def patchify(pixels: torch.Tensor, S: int, P: int) -> torch.Tensor:
    F, g = pixels.shape[0], S // P
    x = pixels.reshape(F, 3, g, P, g, P).permute(0, 2, 4, 1, 3, 5)
    return _b(x.reshape(F * g * g, 3 * P * P).to(F64))


def frame_attention(q, k, v, scale):
    """Intra-frame attention, q/k/v [f, heads, T, hd] (T.attention with the
    block-diagonal mask)."""
    s = (q @ k.transpose(-1, -2)) * scale
    m = s.amax(-1, keepdim=True)
    pr = torch.exp(s - m)
    pr = pr / pr.sum(-1, keepdim=True)
    return pr @ v


def vision_forward(c: T.Cfg, W, pixels, dev, frame_chunk: int = 16) -> torch.Tensor:
    """Frames [F, 3*S*S] -> projector embeddings [F*T, dim] (bf16-valued float64)."""
    pixels = torch.as_tensor(np.asarray(pixels, dtype=np.float32)).to(dev)
    F, Tt, vd, hd, nh = pixels.shape[0], c.T, c.v_dim, c.v_head_dim, c.v_heads
    out = torch.empty(F * Tt, c.dim, dtype=F64, device=dev)
    scale = 1.0 / math.sqrt(hd)
    for f0 in range(0, F, frame_chunk):
        f1 = min(F, f0 + frame_chunk)
        n = (f1 - f0) * Tt
        x = patchify(pixels[f0:f1], c.image_size, c.patch)
        h = _s(W["pos"].repeat(f1 - f0, 1) + linear(x, W["patch_w"], W["patch_b"]))
        for l in range(c.v_layers):
            p = f"vision.{l}."
            xn = layernorm(h, W[p + "ln1_w"], W[p + "ln1_b"], c.ln_eps)
            qkv = _b(linear(xn, W[p + "wqkv"], W[p + "bqkv"]))
            q, k, v = (qkv[:, i * vd:(i + 1) * vd].reshape(f1 - f0, Tt, nh, hd).transpose(1, 2)
                       for i in range(3))  # [f, h, T, hd]
            o = _b(frame_attention(q, k, v, scale).transpose(1, 2).reshape(n, vd))
            h = _s(h + linear(o, W[p + "wo"], W[p + "bo"]))
            xn = layernorm(h, W[p + "ln2_w"], W[p + "ln2_b"], c.ln_eps)
            mid = _b(gelu_tanh(linear(xn, W[p + "w1"], W[p + "b1"])))
            h = _s(h + linear(mid, W[p + "w2"], W[p + "b2"]))
        xn = layernorm(h, W["post_w"], W["post_b"], c.ln_eps)
        p1 = _b(gelu_tanh(linear(xn, W["p1_w"], W["p1_b"])))
        out[f0 * Tt:f1 * Tt] = _b(linear(p1, W["p2_w"], W["p2_b"]))
    return out


# -------------------------------------------------------------------- stage 2
def rope_tables(c: T.Cfg, pos: np.ndarray, dev):
    cos, sin = T.rope_tables(c, pos)
    return torch.from_numpy(cos).to(dev, F64), torch.from_numpy(sin).to(dev, F64)


def apply_rope(x, cos, sin):
    x1, x2 = x[..., :64], x[..., 64:]
    cc, ss = cos[:, None, :], sin[:, None, :]
    return _b(torch.cat([x1 * cc - x2 * ss, x2 * cc + x1 * ss], -1))


def _attention(q, k, v, Lp: int, Lmax: int, dev, q_block: int = 512):
    """q [L, nq, hd], k/v [L, nkv, hd] -> o [L, nq*hd] (bf16-valued), the MR-SP mask
    of T.mrsp_mask, float64 softmax normalised before the P.V product (as T.attention)."""
    L, nq, hd = q.shape
    nkv = k.shape[1]
    rep = nq // nkv
    scale = 1.0 / math.sqrt(hd)
    o = torch.empty(L, nq * hd, dtype=F64, device=dev)
    ar = torch.arange(L, device=dev)
    row = torch.where(ar >= Lp, (ar - Lp) // max(Lmax, 1), torch.full_like(ar, -1))
    for q0 in range(0, L, q_block):
        q1 = min(L, q0 + q_block)
        kq = ar[q0:q1][:, None]
        kk = ar[None, :q1]
        mask = (kk <= kq) & ((kk < Lp) | (row[None, :q1] == row[q0:q1][:, None]))
        for j in range(nkv):
            qh = q[q0:q1, j * rep:(j + 1) * rep].transpose(0, 1)  # [rep, B, hd]
            s = (qh @ k[:q1, j].T) * scale                         # [rep, B, q1]
            s = s.masked_fill(~mask[None], float("-inf"))
            m = s.amax(-1, keepdim=True)
            pr = torch.exp(s - m)
            pr = pr / pr.sum(-1, keepdim=True)
            oh = pr @ v[:q1, j]                                    # [rep, B, hd]
            o[q0:q1, j * rep * hd:(j + 1) * rep * hd] = oh.transpose(0, 1).reshape(q1 - q0, rep * hd)
            del s, pr
    return _b(o)


def llm_logprobs(c: T.Cfg, seed: int, prefix: str, frame_emb: torch.Tensor, question, resp,
                 lengths, dev, row_chunk: int = 8192, vocab_chunk: int = 16384,
                 q_block: int = 512, return_hidden: bool = False):
    """T.llm_logprobs: per-token log-probs (and lse) of the response tokens,
    row-major over (g, j < len_g), as float64 numpy arrays."""
    n_frame_tok = frame_emb.shape[0]
    tok, pos, pad, Lp, L = T.pack(n_frame_tok, question, resp, lengths)
    resp = np.asarray(resp)
    G, Lmax = resp.shape
    d, hd, nq, nkv = c.dim, c.head_dim, c.n_q_heads, c.n_kv_heads
    h = torch.empty(L, d, dtype=F64, device=dev)
    h[:n_frame_tok] = frame_emb.to(dev, F64)
    txt = tok[n_frame_tok:]
    uniq, inv = np.unique(txt, return_inverse=True)
    emb_rows = init_bf16((c.vocab, d), seed, prefix + "embed", T.K_EMBED, dev, rows=uniq)
    h[n_frame_tok:] = emb_rows[torch.from_numpy(inv.reshape(-1)).to(dev)]
    cos, sin = rope_tables(c, pos, dev)
    for l in range(c.layers):
        W = llm_layer_weights(c, seed, prefix, l, dev)
        qkv = torch.empty(L, (nq + 2 * nkv) * hd, dtype=F64, device=dev)
        for r0 in range(0, L, row_chunk):
            r1 = min(L, r0 + row_chunk)
            xn = rmsnorm(h[r0:r1], W["attn_norm"], c.rms_eps)
            qkv[r0:r1] = _b(linear(xn, W["wqkv"], W["bqkv"]))
        q = apply_rope(qkv[:, :nq * hd].reshape(L, nq, hd), cos, sin)
        k = apply_rope(qkv[:, nq * hd:(nq + nkv) * hd].reshape(L, nkv, hd), cos, sin)
        v = qkv[:, (nq + nkv) * hd:].reshape(L, nkv, hd).contiguous()
        del qkv
        o = _attention(q, k, v, Lp, Lmax, dev, q_block)
        del q, k, v
        for r0 in range(0, L, row_chunk):
            r1 = min(L, r0 + row_chunk)
            hh = _s(h[r0:r1] + linear(o[r0:r1], W["wo"]))
            xn = rmsnorm(hh, W["mlp_norm"], c.rms_eps)
            g_ = _s(linear(xn, W["w_gate"]))
            u_ = _s(linear(xn, W["w_up"]))
            act = _b(silu(g_) * u_)
            del g_, u_
            h[r0:r1] = _s(hh + linear(act, W["w_down"]))
        del o, W
    rows, tgts = [], []
    for g in range(G):
        for j in range(int(lengths[g])):
            rows.append(Lp + g * Lmax + j)
            tgts.append(int(resp[g, j]))
    S = len(rows)
    xs = rmsnorm(h[torch.as_tensor(rows, dtype=torch.int64, device=dev)],
                 init_f32((d,), seed, prefix + "final_norm", T.K_NORM, 1.0, dev), c.rms_eps)
    tg = torch.as_tensor(tgts, dtype=torch.int64, device=dev)
    m = torch.full((S,), float("-inf"), dtype=F64, device=dev)
    tl = torch.zeros(S, dtype=F64, device=dev)
    chunks = []
    key_name = prefix + "lm_head"
    for v0 in range(0, c.vocab, vocab_chunk):
        v1 = min(c.vocab, v0 + vocab_chunk)
        wl = init_bf16((c.vocab, d), seed, key_name, T.wscale(d), dev, rows=np.arange(v0, v1))
        lg = xs @ wl.T                                            # [S, v1 - v0]
        m = torch.maximum(m, lg.amax(-1))
        sel = (tg >= v0) & (tg < v1)
        tl[sel] = lg[sel, tg[sel] - v0]
        chunks.append((v0, v1))
    ssum = torch.zeros(S, dtype=F64, device=dev)
    for v0, v1 in chunks:  # second pass: the max-shifted sum (exact two-pass LSE, as numpy)
        wl = init_bf16((c.vocab, d), seed, key_name, T.wscale(d), dev, rows=np.arange(v0, v1))
        ssum += torch.exp(xs @ wl.T - m[:, None]).sum(-1)
    lse = m + torch.log(ssum)
    lp = (tl - lse).cpu().numpy()
    out = (lp, lse.cpu().numpy())
    return out + (h,) if return_hidden else out
