"""CPU oracle for the transformer-shaped MR-SP path — TEST INFRASTRUCTURE.

Imported only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs; never by the product package.

Parity status: PINNED. Conventions to the reference (below); arithmetic to
the published implementations of both model families — with storage rounding
off (`exact()`), vision_forward matches HF transformers' SiglipVisionModel
(+ an mlp2x_gelu projector) to 2e-15 and llm_logprobs matches
Qwen2ForCausalLM to 4e-15 in float64 (2e-7 against stock HF, whose RMSNorm
statistic and RoPE cos/sin are float32), at c1 and at production widths
(tests/test_oracle_hf_pin.py). The RoPE inverse frequencies follow HF's
float32 formula (rope_inv_freq).

The reference (lvrl, /root/reference/proj) has no transformer: its "vision
tower" is tanh(Wx) (policy.cpp:36-47) and its "LLM" a pooled-context MLP
(policy.cpp:85-119). This restatement keeps every contract the reference fixes
and that the tests pin bit-exactly elsewhere —
  * frames from gen_video (mmseq.cpp:58-72) and the shard plans (engine.cpp:15-29),
  * prompt = [frame embeddings | question] (build_sequence, mmseq.cpp:139-151),
    shared by the G rollouts (context_vector replicated, grpo.cpp:53),
  * rows padded with PAD=0 to the longest rollout (pad_batch, engine.cpp:31-43),
  * teacher forcing with prev = EOS at t = 0 (engine.cpp:124, policy.cpp:127),
  * max-shifted log-softmax then gather lp[y] (common.hpp:95-104, grpo.cpp:82-85)
— and restates the SigLIP-/Qwen2.5-shaped arithmetic the north star asks for
(BASELINE.json) in float64 over bf16-rounded weights/inputs, rounding to bf16
at exactly the tensor boundaries where the device stores bf16.

Weights: the engine's counter-based init (csrc/engine.cu:init_weights),
    key = splitmix64(seed ^ fnv1a64(name)),
    u_i = (splitmix64(key + i) >> 40) * 2^-24,
    w_i = bf16(fp32(a) * (2 u_i - 1))            (bf16 tensors)
    w_i = fp32(offset + fp32(a) * (2 u_i - 1))   (fp32 tensors)
is reproduced bit-for-bit here (tests/test_transformer_oracle.py).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Dict

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


# --------------------------------------------------------------------------- RNG
def _splitmix_np(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _splitmix_int(z: int) -> int:
    return int(_splitmix_np(np.array([z & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64))[0])


def fnv1a64(s: str) -> int:
    h = 1469598103934665603
    for c in s.encode():
        h ^= c
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def tensor_key(seed: int, name: str) -> int:
    return _splitmix_int(seed ^ fnv1a64(name))


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round float32 -> bf16 (round to nearest even), returned as float32."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    b = x.view(np.uint32).astype(np.uint64)
    b = (b + ((b >> np.uint64(16)) & np.uint64(1)) + np.uint64(0x7FFF)) & np.uint64(0xFFFF0000)
    return b.astype(np.uint32).view(np.float32)


def _uniform_t(n: int, key: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        idx = np.arange(n, dtype=np.uint64) + np.uint64(key)
    u = (_splitmix_np(idx) >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -24)
    return np.float32(2.0) * u - np.float32(1.0)


def init_bf16(shape, seed: int, name: str, a: float) -> np.ndarray:
    n = int(np.prod(shape))
    return bf16_round(np.float32(a) * _uniform_t(n, tensor_key(seed, name))).reshape(shape)


def init_f32(shape, seed: int, name: str, a: float, offset: float) -> np.ndarray:
    n = int(np.prod(shape))
    t = np.float32(a) * _uniform_t(n, tensor_key(seed, name))
    return (np.float32(offset) + t).astype(np.float32).reshape(shape)


def wscale(fan_in: int) -> float:
    return float(np.float32(math.sqrt(3.0 / fan_in)))


K_BIAS, K_NORM, K_POS, K_EMBED = 0.03, 0.1, 0.1, float(np.float32(math.sqrt(3.0)))


# ------------------------------------------------------------------ model config
@dataclass
class Cfg:
    image_size: int
    patch: int
    v_dim: int
    v_heads: int
    v_head_dim: int
    v_mlp: int
    v_layers: int
    dim: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    mlp: int
    layers: int
    vocab: int
    rope_theta: float = 1e6
    rms_eps: float = 1e-6
    ln_eps: float = 1e-6

    @property
    def T(self) -> int:
        return (self.image_size // self.patch) ** 2

    @classmethod
    def from_any(cls, c) -> "Cfg":
        if isinstance(c, cls):
            return c
        d = c.as_dict() if hasattr(c, "as_dict") else dict(c)
        return cls(**{k: d[k] for k in cls.__dataclass_fields__})


def vision_weights(c: Cfg, seed: int) -> Dict[str, np.ndarray]:
    kreal = 3 * c.patch * c.patch
    vd = c.v_dim
    W = {
        "patch_w": init_bf16((vd, kreal), seed, "vision.patch_w", wscale(kreal)),
        "patch_b": init_f32((vd,), seed, "vision.patch_b", K_BIAS, 0.0),
        "pos": init_f32((c.T, vd), seed, "vision.pos", K_POS, 0.0),
        "post_w": init_f32((vd,), seed, "vision.post_w", K_NORM, 1.0),
        "post_b": init_f32((vd,), seed, "vision.post_b", K_BIAS, 0.0),
        "p1_w": init_bf16((c.dim, vd), seed, "proj.w1", wscale(vd)),
        "p1_b": init_f32((c.dim,), seed, "proj.b1", K_BIAS, 0.0),
        "p2_w": init_bf16((c.dim, c.dim), seed, "proj.w2", wscale(c.dim)),
        "p2_b": init_f32((c.dim,), seed, "proj.b2", K_BIAS, 0.0),
    }
    for l in range(c.v_layers):
        p = f"vision.{l}."
        W[p + "ln1_w"] = init_f32((vd,), seed, p + "ln1_w", K_NORM, 1.0)
        W[p + "ln1_b"] = init_f32((vd,), seed, p + "ln1_b", K_BIAS, 0.0)
        W[p + "wqkv"] = init_bf16((3 * vd, vd), seed, p + "wqkv", wscale(vd))
        W[p + "bqkv"] = init_f32((3 * vd,), seed, p + "bqkv", K_BIAS, 0.0)
        W[p + "wo"] = init_bf16((vd, vd), seed, p + "wo", wscale(vd))
        W[p + "bo"] = init_f32((vd,), seed, p + "bo", K_BIAS, 0.0)
        W[p + "ln2_w"] = init_f32((vd,), seed, p + "ln2_w", K_NORM, 1.0)
        W[p + "ln2_b"] = init_f32((vd,), seed, p + "ln2_b", K_BIAS, 0.0)
        W[p + "w1"] = init_bf16((c.v_mlp, vd), seed, p + "w1", wscale(vd))
        W[p + "b1"] = init_f32((c.v_mlp,), seed, p + "b1", K_BIAS, 0.0)
        W[p + "w2"] = init_bf16((vd, c.v_mlp), seed, p + "w2", wscale(c.v_mlp))
        W[p + "b2"] = init_f32((vd,), seed, p + "b2", K_BIAS, 0.0)
    return W


def llm_weights(c: Cfg, seed: int, prefix: str) -> Dict[str, np.ndarray]:
    d, hd = c.dim, c.head_dim
    qkv_rows = (c.n_q_heads + 2 * c.n_kv_heads) * hd
    W = {"embed": init_bf16((c.vocab, d), seed, prefix + "embed", K_EMBED),
         "final_norm": init_f32((d,), seed, prefix + "final_norm", K_NORM, 1.0),
         "lm_head": init_bf16((c.vocab, d), seed, prefix + "lm_head", wscale(d))}
    for l in range(c.layers):
        p = f"{prefix}{l}."
        W[f"{l}.attn_norm"] = init_f32((d,), seed, p + "attn_norm", K_NORM, 1.0)
        W[f"{l}.wqkv"] = init_bf16((qkv_rows, d), seed, p + "wqkv", wscale(d))
        W[f"{l}.bqkv"] = init_f32((qkv_rows,), seed, p + "bqkv", K_BIAS, 0.0)
        W[f"{l}.wo"] = init_bf16((d, c.n_q_heads * hd), seed, p + "wo", wscale(c.n_q_heads * hd))
        W[f"{l}.mlp_norm"] = init_f32((d,), seed, p + "mlp_norm", K_NORM, 1.0)
        W[f"{l}.w_gate"] = init_bf16((c.mlp, d), seed, p + "w_gate", wscale(d))
        W[f"{l}.w_up"] = init_bf16((c.mlp, d), seed, p + "w_up", wscale(d))
        W[f"{l}.w_down"] = init_bf16((d, c.mlp), seed, p + "w_down", wscale(c.mlp))
    return W


# -------------------------------------------------------------------- pieces
def _f64(x):
    return np.asarray(x, dtype=np.float64)


# Storage rounding. The device stores bf16 activations and an fp32 residual
# stream; the oracle rounds at exactly those tensor boundaries. Inside
# `exact()` both are the identity: the same algorithm in plain float64, which
# is what tests/test_oracle_hf_pin.py compares with the published
# implementations (HF transformers SigLIP / Qwen2) to pin the conventions.
_EXACT = [False]


def _b(x):
    """bf16 storage (fp32 then round-to-nearest-even bf16)."""
    return _f64(x) if _EXACT[0] else bf16_round(np.asarray(x).astype(np.float32))


def _s(x):
    """fp32 storage."""
    return _f64(x) if _EXACT[0] else np.asarray(x).astype(np.float32)


class exact:
    """Context manager: the oracle's algorithm without storage rounding."""

    def __enter__(self):
        self._old = _EXACT[0]
        _EXACT[0] = True
        return self

    def __exit__(self, *a):
        _EXACT[0] = self._old


def layernorm(x, w, b, eps):
    x = _f64(x)
    mu = x.mean(-1, keepdims=True)
    var = ((x - mu) ** 2).mean(-1, keepdims=True)
    return _b((x - mu) / np.sqrt(var + eps) * w + b)


def rmsnorm(x, w, eps):
    x = _f64(x)
    r = 1.0 / np.sqrt((x * x).mean(-1, keepdims=True) + eps)
    return _b(w * (x * r))


def gelu_tanh(x):
    return 0.5 * x * (1.0 + np.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))


def silu(x):
    return x / (1.0 + np.exp(-x))


def linear(x, w, b=None):
    y = _f64(x) @ _f64(w).T
    return y if b is None else y + b


def patchify(pixels: np.ndarray, S: int, P: int) -> np.ndarray:
    """[F, 3*S*S] -> [F*T, 3*P*P], column c*P*P + ky*P + kx (conv weight layout)."""
    F = pixels.shape[0]
    g = S // P
    x = pixels.reshape(F, 3, g, P, g, P).transpose(0, 2, 4, 1, 3, 5)
    return _b(x.reshape(F * g * g, 3 * P * P))


def attention(q, k, v, mask, scale):
    """q [nq, L, hd], k/v [nkv, L, hd] float64; GQA by head grouping."""
    rep = q.shape[0] // k.shape[0]
    k = np.repeat(k, rep, 0)
    v = np.repeat(v, rep, 0)
    s = np.einsum("hqd,hkd->hqk", q, k) * scale
    s = np.where(mask[None], s, -np.inf)
    m = s.max(-1, keepdims=True)
    m = np.where(np.isfinite(m), m, 0.0)
    p = np.exp(s - m)
    p /= np.maximum(p.sum(-1, keepdims=True), 1e-300)
    return np.einsum("hqk,hkd->hqd", p, v)


def mrsp_mask(L: int, Lp: int, Lmax: int) -> np.ndarray:
    """k <= q and (k < Lp or row(k) == row(q)) — see csrc/attention.cu."""
    q = np.arange(L)[:, None]
    k = np.arange(L)[None, :]
    rq = np.where(q >= Lp, (q - Lp) // max(Lmax, 1), -1)
    rk = np.where(k >= Lp, (k - Lp) // max(Lmax, 1), -2)
    return (k <= q) & ((k < Lp) | (rq == rk))


# -------------------------------------------------------------------- stage 1
def vision_forward(c: Cfg, W, pixels: np.ndarray) -> np.ndarray:
    """Frames [F, 3*S*S] -> projector embeddings [F*T, dim] (bf16-valued)."""
    F = pixels.shape[0]
    T, vd, hd = c.T, c.v_dim, c.v_head_dim
    x = patchify(pixels, c.image_size, c.patch)
    h = _s(np.tile(_f64(W["pos"]), (F, 1)) + linear(x, W["patch_w"], W["patch_b"]))
    blk = np.kron(np.eye(F, dtype=bool), np.ones((T, T), dtype=bool))
    for l in range(c.v_layers):
        p = f"vision.{l}."
        xn = layernorm(h, W[p + "ln1_w"], W[p + "ln1_b"], c.ln_eps)
        qkv = _b(linear(xn, W[p + "wqkv"], W[p + "bqkv"]))
        n = qkv.shape[0]
        q = _f64(qkv[:, :vd]).reshape(n, c.v_heads, hd).transpose(1, 0, 2)
        k = _f64(qkv[:, vd:2 * vd]).reshape(n, c.v_heads, hd).transpose(1, 0, 2)
        v = _f64(qkv[:, 2 * vd:]).reshape(n, c.v_heads, hd).transpose(1, 0, 2)
        o = attention(q, k, v, blk, 1.0 / math.sqrt(hd)).transpose(1, 0, 2).reshape(n, vd)
        o = _b(o)
        h = _s(h + linear(o, W[p + "wo"], W[p + "bo"]))
        xn = layernorm(h, W[p + "ln2_w"], W[p + "ln2_b"], c.ln_eps)
        mid = _b(gelu_tanh(linear(xn, W[p + "w1"], W[p + "b1"])))
        h = _s(h + linear(mid, W[p + "w2"], W[p + "b2"]))
    xn = layernorm(h, W["post_w"], W["post_b"], c.ln_eps)
    p1 = _b(gelu_tanh(linear(xn, W["p1_w"], W["p1_b"])))
    return _b(linear(p1, W["p2_w"], W["p2_b"]))


# -------------------------------------------------------------------- stage 2
def pack(n_frame_tok: int, question, resp, lengths):
    """Packed layout (mrsp_op_pack_sequence): tokens (-1 at frame positions),
    position ids and pad mask for [frames | question | G x Lmax]."""
    question = np.asarray(question)
    G, Lmax = resp.shape
    Lp = n_frame_tok + len(question)
    L = Lp + G * Lmax
    tok = np.full(L, -1, dtype=np.int64)
    tok[n_frame_tok:Lp] = question
    pos = np.arange(L, dtype=np.int64)
    pad = np.zeros(L, dtype=np.uint8)
    for g in range(G):
        base = Lp + g * Lmax
        pos[base:base + Lmax] = Lp + np.arange(Lmax)
        ln = int(lengths[g])
        row = np.zeros(Lmax, dtype=np.int64)  # PAD
        if ln > 0:
            row[0] = 1  # EOS: prev token at t = 0 (engine.cpp:124)
            row[1:ln] = resp[g, : ln - 1]
        pad[base + ln: base + Lmax] = 1
        tok[base:base + Lmax] = row
    return tok, pos, pad, Lp, L


def rope_inv_freq(theta: float) -> np.ndarray:
    """inv_freq[i] = 1 / theta^(2i/128) in float32, as HF transformers builds it
    (`1.0 / (base ** (torch.arange(0, dim, 2).float() / dim))`, Qwen2
    RotaryEmbedding): the exponent and the power are float32, the power
    correctly rounded (torch's CPU powf can differ by 1 ulp in one entry of 64
    for theta = 1e6; tests/test_oracle_hf_pin.py bounds that)."""
    e = np.arange(0, 128, 2).astype(np.float32) / np.float32(128.0)
    a = np.power(np.float64(np.float32(theta)), e.astype(np.float64)).astype(np.float32)
    return (np.float32(1.0) / a).astype(np.float32)


def rope_tables(c: Cfg, pos: np.ndarray):
    """cos/sin of the fp32 angle pos * inv_freq (fp32 product, as HF and the
    device compute it), each rounded to fp32."""
    inv = rope_inv_freq(c.rope_theta)
    ang = pos.astype(np.float32)[:, None] * inv[None, :]  # fp32 product (as the device)
    return np.cos(_f64(ang)).astype(np.float32), np.sin(_f64(ang)).astype(np.float32)


def apply_rope(x: np.ndarray, cos, sin) -> np.ndarray:
    """x [L, H, 128] bf16-valued -> bf16 (rotate-half)."""
    x1, x2 = _f64(x[..., :64]), _f64(x[..., 64:])
    c, s = _f64(cos[:, None, :]), _f64(sin[:, None, :])
    return _b(np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], -1))


def llm_logprobs(c: Cfg, W, frame_emb, question, resp, lengths, return_hidden=False):
    """Per-token log-probs of the response tokens (row-major over (g, j < len_g))."""
    n_frame_tok = frame_emb.shape[0]
    tok, pos, pad, Lp, L = pack(n_frame_tok, question, resp, lengths)
    G, Lmax = resp.shape
    d, hd, nq, nkv = c.dim, c.head_dim, c.n_q_heads, c.n_kv_heads
    h = np.empty((L, d), dtype=np.float64 if _EXACT[0] else np.float32)
    h[:n_frame_tok] = frame_emb
    h[n_frame_tok:] = W["embed"][tok[n_frame_tok:]]
    cos, sin = rope_tables(c, pos)
    mask = mrsp_mask(L, Lp, Lmax)
    for l in range(c.layers):
        xn = rmsnorm(h, W[f"{l}.attn_norm"], c.rms_eps)
        qkv = _b(linear(xn, W[f"{l}.wqkv"], W[f"{l}.bqkv"]))
        q = apply_rope(qkv[:, : nq * hd].reshape(L, nq, hd), cos, sin)
        k = apply_rope(qkv[:, nq * hd:(nq + nkv) * hd].reshape(L, nkv, hd), cos, sin)
        v = qkv[:, (nq + nkv) * hd:].reshape(L, nkv, hd)
        o = attention(_f64(q).transpose(1, 0, 2), _f64(k).transpose(1, 0, 2),
                      _f64(v).transpose(1, 0, 2), mask, 1.0 / math.sqrt(hd))
        o = _b(o.transpose(1, 0, 2).reshape(L, nq * hd))
        h = _s(h + linear(o, W[f"{l}.wo"]))
        xn = rmsnorm(h, W[f"{l}.mlp_norm"], c.rms_eps)
        g_ = _s(linear(xn, W[f"{l}.w_gate"]))
        u_ = _s(linear(xn, W[f"{l}.w_up"]))
        act = _b(silu(_f64(g_)) * u_)
        h = _s(h + linear(act, W[f"{l}.w_down"]))
    rows, tgts = [], []
    for g in range(G):
        for j in range(int(lengths[g])):
            rows.append(Lp + g * Lmax + j)
            tgts.append(int(resp[g, j]))
    xs = rmsnorm(h[rows], W["final_norm"], c.rms_eps)
    logits = linear(xs, W["lm_head"])
    m = logits.max(-1, keepdims=True)
    lse = (m + np.log(np.exp(logits - m).sum(-1, keepdims=True)))[:, 0]
    lp = logits[np.arange(len(rows)), tgts] - lse
    if return_hidden:
        return lp, lse, h
    return lp, lse


# ------------------------------------------------------------- FLOP accounting
def step_flops(c: Cfg, frames: int, n_q: int, lengths, passes: int = 2) -> dict:
    """Algorithmic FLOPs of one MR-SP step (SURVEY §8d formulas; pads excluded,
    shared prefix counted once per pass)."""
    T, vd, hd = c.T, c.v_dim, c.v_head_dim
    kreal = 3 * c.patch * c.patch
    per_frame = (2 * T * c.v_layers * (4 * vd * vd + 2 * vd * c.v_mlp)
                 + c.v_layers * 4 * T * T * vd + 2 * T * kreal * vd
                 + 2 * T * (vd * c.dim + c.dim * c.dim))
    Lp = frames * T + n_q
    S = int(np.sum(lengths))
    d, nq, nkv, mlp, L = c.dim, c.n_q_heads, c.n_kv_heads, c.mlp, c.layers
    lin_tok = 2 * L * (d * (nq * c.head_dim + 2 * nkv * c.head_dim) + nq * c.head_dim * d + 3 * d * mlp)
    lin = lin_tok * (Lp + S)
    attn_prefix = 2 * L * nq * c.head_dim * Lp * Lp
    attn_resp = sum(4 * L * nq * c.head_dim * int(l) * (Lp + int(l) / 2) for l in lengths)
    lm = 2 * d * c.vocab * S
    per_pass = lin + attn_prefix + attn_resp + lm
    return {"encode": per_frame * frames, "linear": lin, "attn_prefix": attn_prefix,
            "attn_resp": attn_resp, "lm_head": lm, "per_pass": per_pass,
            "step": per_frame * frames + passes * per_pass, "tokens": Lp + S, "Lp": Lp, "scored": S}
