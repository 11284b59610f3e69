"""CPU: pins the transformer oracle (oracle/transformer.py) to the published
implementations of the two model families it restates — HF transformers'
SigLIP vision tower (SiglipVisionModel) and Qwen2 decoder (Qwen2ForCausalLM)
— run in float64 on the oracle's own weights.

The oracle's storage rounding (bf16 activations, fp32 residual) is switched
off (`T.exact()`), so both sides compute the same algorithm in plain float64
and any convention difference (RoPE layout or frequencies, GELU variant,
LayerNorm/RMSNorm eps placement, GQA head grouping, attention scale, q/k/v
split, projector order, teacher-forcing mask) shows up as an O(1e-2..1)
error instead of hiding under bf16 noise. Measured: vision embeddings agree
to 2e-15 relative; per-token log-probs to 2e-7 against stock HF, whose
RMSNorm statistic and RoPE cos/sin are float32 islands, and to 4e-15 once
those two steps are lifted to float64 (`hf_float64_upcasts`: same formulas).

The projector has no HF class: it is LLaVA's mlp2x_gelu layout (Linear,
GELU, Linear) with the tanh GELU, built from torch.nn.

Anchors: the teacher-forcing and log-softmax conventions the oracle shares
with the reference (policy.cpp:159-174, grpo.cpp:82-85, common.hpp:95-104);
SURVEY §8c.
"""
import numpy as np
import pytest
import torch

from oracle import transformer as T
from paper_2507_07966_b200 import engine as E

transformers = pytest.importorskip("transformers")


def _t(x):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64)))


def hf_vision(c: T.Cfg, W):
    """SiglipVisionModel + mlp2x_gelu projector holding the oracle's weights."""
    from transformers import SiglipVisionConfig, SiglipVisionModel
    cfg = SiglipVisionConfig(hidden_size=c.v_dim, intermediate_size=c.v_mlp,
                             num_hidden_layers=c.v_layers, num_attention_heads=c.v_heads,
                             num_channels=3, image_size=c.image_size, patch_size=c.patch,
                             hidden_act="gelu_pytorch_tanh", layer_norm_eps=c.ln_eps,
                             attention_dropout=0.0, vision_use_head=False)
    cfg._attn_implementation = "sdpa"  # float64 softmax (eager upcasts to float32)
    tower = SiglipVisionModel(cfg).double().eval()
    vd, P = c.v_dim, c.patch
    sd = {
        "vision_model.embeddings.patch_embedding.weight": _t(W["patch_w"]).reshape(vd, 3, P, P),
        "vision_model.embeddings.patch_embedding.bias": _t(W["patch_b"]),
        "vision_model.embeddings.position_embedding.weight": _t(W["pos"]),
        "vision_model.post_layernorm.weight": _t(W["post_w"]),
        "vision_model.post_layernorm.bias": _t(W["post_b"]),
    }
    for l in range(c.v_layers):
        p, h = f"vision.{l}.", f"vision_model.encoder.layers.{l}."
        wqkv, bqkv = _t(W[p + "wqkv"]), _t(W[p + "bqkv"])
        for i, n in enumerate(("q_proj", "k_proj", "v_proj")):  # rows [q | k | v]
            sd[h + f"self_attn.{n}.weight"] = wqkv[i * vd:(i + 1) * vd]
            sd[h + f"self_attn.{n}.bias"] = bqkv[i * vd:(i + 1) * vd]
        sd[h + "self_attn.out_proj.weight"] = _t(W[p + "wo"])
        sd[h + "self_attn.out_proj.bias"] = _t(W[p + "bo"])
        for a, b in (("layer_norm1", "ln1"), ("layer_norm2", "ln2")):
            sd[h + f"{a}.weight"] = _t(W[p + b + "_w"])
            sd[h + f"{a}.bias"] = _t(W[p + b + "_b"])
        sd[h + "mlp.fc1.weight"], sd[h + "mlp.fc1.bias"] = _t(W[p + "w1"]), _t(W[p + "b1"])
        sd[h + "mlp.fc2.weight"], sd[h + "mlp.fc2.bias"] = _t(W[p + "w2"]), _t(W[p + "b2"])
    missing, unexpected = tower.load_state_dict(sd, strict=False)
    assert not unexpected and all("position_ids" in k for k in missing), (missing, unexpected)
    proj = torch.nn.Sequential(torch.nn.Linear(vd, c.dim), torch.nn.GELU(approximate="tanh"),
                               torch.nn.Linear(c.dim, c.dim)).double()
    proj.load_state_dict({"0.weight": _t(W["p1_w"]), "0.bias": _t(W["p1_b"]),
                          "2.weight": _t(W["p2_w"]), "2.bias": _t(W["p2_b"])})

    def run(pixels):
        F = pixels.shape[0]
        x = _t(pixels).reshape(F, 3, c.image_size, c.image_size)
        with torch.no_grad():
            feats = tower(pixel_values=x).last_hidden_state  # [F, T, vd], post-LN
            return proj(feats).reshape(F * c.T, c.dim).numpy()
    return run


def hf_llm(c: T.Cfg, W):
    """Qwen2ForCausalLM holding the oracle's LLM weights."""
    from transformers import Qwen2Config, Qwen2ForCausalLM
    hd, nq, nkv = c.head_dim, c.n_q_heads, c.n_kv_heads
    cfg = Qwen2Config(vocab_size=c.vocab, hidden_size=c.dim, intermediate_size=c.mlp,
                      num_hidden_layers=c.layers, num_attention_heads=nq,
                      num_key_value_heads=nkv, head_dim=hd, rope_theta=c.rope_theta,
                      rms_norm_eps=c.rms_eps, tie_word_embeddings=False,
                      max_position_embeddings=1 << 20, use_sliding_window=False,
                      attention_dropout=0.0)
    cfg._attn_implementation = "sdpa"
    m = Qwen2ForCausalLM(cfg).double().eval()
    sd = {"model.embed_tokens.weight": _t(W["embed"]), "model.norm.weight": _t(W["final_norm"]),
          "lm_head.weight": _t(W["lm_head"])}
    for l in range(c.layers):
        h = f"model.layers.{l}."
        wqkv, bqkv = _t(W[f"{l}.wqkv"]), _t(W[f"{l}.bqkv"])
        cuts = [0, nq * hd, (nq + nkv) * hd, (nq + 2 * nkv) * hd]
        for i, n in enumerate(("q_proj", "k_proj", "v_proj")):
            sd[h + f"self_attn.{n}.weight"] = wqkv[cuts[i]:cuts[i + 1]]
            sd[h + f"self_attn.{n}.bias"] = bqkv[cuts[i]:cuts[i + 1]]
        sd[h + "self_attn.o_proj.weight"] = _t(W[f"{l}.wo"])
        sd[h + "input_layernorm.weight"] = _t(W[f"{l}.attn_norm"])
        sd[h + "post_attention_layernorm.weight"] = _t(W[f"{l}.mlp_norm"])
        sd[h + "mlp.gate_proj.weight"] = _t(W[f"{l}.w_gate"])
        sd[h + "mlp.up_proj.weight"] = _t(W[f"{l}.w_up"])
        sd[h + "mlp.down_proj.weight"] = _t(W[f"{l}.w_down"])
    missing, unexpected = m.load_state_dict(sd, strict=False)
    assert not missing and not unexpected, (missing, unexpected)
    return m


def hf_logprobs(c: T.Cfg, m, frame_emb, grp):
    """Packed [frames | question | G x Lmax] sequence through Qwen2 with the
    MR-SP mask as a 4D attention mask and the oracle's position ids; per-token
    log-probs of the scored positions (teacher forcing, prev = EOS at t = 0)."""
    tok, pos, pad, Lp, L = T.pack(frame_emb.shape[0], grp.question, grp.resp, grp.lengths)
    nf = frame_emb.shape[0]
    with torch.no_grad():
        emb = m.model.embed_tokens.weight
        x = torch.cat([_t(frame_emb), emb[torch.from_numpy(tok[nf:])]])[None]
        mask = torch.from_numpy(T.mrsp_mask(L, Lp, grp.Lmax))[None, None]
        logits = m(inputs_embeds=x, position_ids=torch.from_numpy(pos)[None],
                   attention_mask=mask).logits[0]
        lsm = torch.log_softmax(logits, -1).numpy()
    rows = [Lp + g * grp.Lmax + j for g in range(len(grp.lengths)) for j in range(grp.lengths[g])]
    tg = [int(grp.resp[g, j]) for g in range(len(grp.lengths)) for j in range(grp.lengths[g])]
    return lsm[rows, tg]


def _check_inv_freq(c: T.Cfg, m):
    """The engine/oracle RoPE table is HF's float32 formula: identical except
    where torch's CPU powf misses the correctly rounded power by 1 ulp."""
    hf = m.model.rotary_emb.inv_freq.float().numpy()
    ours = T.rope_inv_freq(c.rope_theta)
    ulps = np.abs(hf.view(np.int32).astype(np.int64) - ours.view(np.int32).astype(np.int64))
    assert ulps.max() <= 1 and (ulps > 0).sum() <= 2, ulps
    # the forward comparison below then isolates everything else
    m.model.rotary_emb.inv_freq.copy_(torch.from_numpy(ours.astype(np.float64)))
    m.model.rotary_emb.original_inv_freq = m.model.rotary_emb.inv_freq.clone()


class hf_float64_upcasts:
    """Lifts HF Qwen2's two float32 islands to float64 — the RMSNorm statistic
    (`hidden_states.to(torch.float32)`) and the cos/sin of the float32 RoPE
    angle (then rounded to float32 as HF does, but from a correctly rounded
    cos/sin). Formulas unchanged; only the precision of those two steps."""

    def __enter__(self):
        from transformers.models.qwen2 import modeling_qwen2 as mq
        self.mq = mq
        self.saved = (mq.Qwen2RMSNorm.forward, mq.Qwen2RotaryEmbedding.forward)

        def rms(mod, h):
            var = h.pow(2).mean(-1, keepdim=True)
            return mod.weight * (h * torch.rsqrt(var + mod.variance_epsilon))

        def rope(mod, x, position_ids):
            ang = position_ids.float()[..., None] * mod.inv_freq.float()  # float32, as HF
            emb = torch.cat((ang, ang), -1).double()
            return (emb.cos().float().to(x.dtype) * mod.attention_scaling,
                    emb.sin().float().to(x.dtype) * mod.attention_scaling)

        mq.Qwen2RMSNorm.forward, mq.Qwen2RotaryEmbedding.forward = rms, rope
        return self

    def __exit__(self, *a):
        self.mq.Qwen2RMSNorm.forward, self.mq.Qwen2RotaryEmbedding.forward = self.saved


def _pin(c: T.Cfg, frames: int, grp, vseed=2, pseed=3, tol_emb=1e-12, tol_lp=1e-6,
         tol_lp_f64=1e-12):
    pix = E.gen_video(5, frames, 3 * c.image_size ** 2)
    Wv = T.vision_weights(c, vseed)
    with T.exact():
        emb = T.vision_forward(c, Wv, pix)
    got = hf_vision(c, Wv)(pix)
    rel = np.linalg.norm(got - emb, axis=1) / np.linalg.norm(emb, axis=1)
    assert rel.max() <= tol_emb, rel.max()
    del Wv
    Wl = T.llm_weights(c, pseed, "policy.")
    # the LLM input is a bf16-valued embedding, as in the engine
    emb16 = T.bf16_round(emb.astype(np.float32))
    with T.exact():
        lp, _ = T.llm_logprobs(c, Wl, emb16, grp.question, grp.resp, grp.lengths)
    m = hf_llm(c, Wl)
    _check_inv_freq(c, m)
    want = hf_logprobs(c, m, emb16, grp)
    d = np.abs(lp - want)
    assert d.max() <= tol_lp, d.max()  # stock HF (float32 RMSNorm statistic / RoPE cos)
    with hf_float64_upcasts():
        want64 = hf_logprobs(c, m, emb16, grp)
    d64 = np.abs(lp - want64)
    assert d64.max() <= tol_lp_f64, d64.max()  # same algorithm to float64 roundoff
    return rel.max(), d.max(), d64.max()


def test_oracle_pinned_to_hf_c1():
    """BASELINE c1 geometry (every layer, both towers)."""
    w = E.workloads()["c1"]
    c = T.Cfg.from_any(w.cfg)
    _pin(c, w.frames, E.make_group(w, seed=3))


def test_oracle_pinned_to_hf_full_width_layer():
    """Production widths: the 27-layer SigLIP-shaped tower (224^2, patch 14,
    16 x 72 heads, MLP 4304) + projector to 3584, and one Qwen2.5-7B-shaped
    decoder layer (28 Q / 4 KV heads x 128, MLP 18944, RoPE theta 1e6). The
    vocabulary is cut to 2048 rows: V only sizes the LM head, it carries no
    convention, and 152064 rows cost minutes of CPU init."""
    w = E.workloads()["c4"]
    d = w.cfg.as_dict()
    d.update(layers=1, vocab=2048)
    c = T.Cfg(**{k: d[k] for k in T.Cfg.__dataclass_fields__})
    wl = E.Workload("pin", E.ModelConfig(**d), 1, 1, 2, 37, 20, 40)
    _pin(c, 1, E.make_group(wl, seed=9))


def test_exact_mode_is_only_storage_rounding():
    """Inside exact() the oracle differs from its default mode by storage
    rounding alone: bf16-level differences, not convention-level ones."""
    w = E.workloads()["c1"]
    c = T.Cfg.from_any(w.cfg)
    pix = E.gen_video(1, w.frames, 3 * c.image_size ** 2)
    Wv = T.vision_weights(c, 2)
    a = T.vision_forward(c, Wv, pix)
    with T.exact():
        b = T.vision_forward(c, Wv, pix)
    rel = np.linalg.norm(a - b, axis=1) / np.linalg.norm(b, axis=1)
    assert 0 < rel.max() <= 2e-2
    assert a.dtype == np.float32 and b.dtype == np.float64
