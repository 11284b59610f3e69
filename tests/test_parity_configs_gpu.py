"""GPU: the benchmarked configurations (BASELINE.json c2, c4) end to end
against the oracle, at SURVEY §8c tolerances.

The engine runs one MR-SP step through the C-ABI (mrsp_engine_step: Stage-1
encode into the cache, G fetches, policy and reference prefill, fused LM-head
log-probs). The oracle is oracle/transformer_torch.py — the float64 twin of
oracle/transformer.py (pinned to it on CPU in tests/test_oracle_twin.py, and
through it to HF SigLIP / Qwen2 in tests/test_oracle_hf_pin.py) — run on the
same device after the engine is closed, from its own counter-generated weights
and its own embeddings (nothing of the engine's state enters the oracle).

Anchors: the reference's at-scale serial-equivalence check
(/root/reference/proj/tests/acceptance.cpp:345-404, serial_prefill at
src/engine.cpp:59-71) and SURVEY §8c: embeddings per-token rel-L2 <= 1e-2 and
cosine >= 0.9995; log-probs max |d| <= 5e-2 and mean |d| <= 5e-3 nats.
"""
import json
import os
import time

import numpy as np
import pytest
import torch

from oracle import transformer as T
from paper_2507_07966_b200 import engine as E

pytestmark = pytest.mark.gpu

VSEED, PSEED, RSEED = 2, 3, 4
EMB_REL, EMB_COS = 1e-2, 0.9995
LP_MAX, LP_MEAN = 5e-2, 5e-3


def _record(name, d):
    out = os.environ.get("MRSP_PARITY_OUT")
    if out:
        with open(out, "a") as f:
            f.write(json.dumps({"case": name, **d}) + "\n")


def _emb_stats(got, want):
    rel = np.linalg.norm(got - want, axis=1) / np.linalg.norm(want, axis=1)
    cos = (got * want).sum(1) / (np.linalg.norm(got, axis=1) * np.linalg.norm(want, axis=1))
    return {"emb_rel_max": float(rel.max()), "emb_rel_mean": float(rel.mean()),
            "emb_cos_min": float(cos.min()), "tokens": int(len(rel))}


def _engine(w, sp, pix, grp, vid):
    eng = E.Engine(w.cfg, sp=sp, vision_seed=VSEED, policy_seed=PSEED, ref_seed=RSEED)
    lp_p, lp_r = eng.step(vid, pix, grp)
    emb = eng.embeddings(vid, w.frames)
    st = eng.stats()
    eng.close()
    return emb, lp_p, lp_r, st


def _oracle(w, pix, grp):
    from oracle import transformer_torch as TT
    c = T.Cfg.from_any(w.cfg)
    t0 = time.time()
    W = TT.vision_weights(c, VSEED, "cuda")
    emb = TT.vision_forward(c, W, pix, "cuda")
    del W
    t1 = time.time()
    lp_p, _ = TT.llm_logprobs(c, PSEED, "policy.", emb, grp.question, grp.resp, grp.lengths, "cuda")
    lp_r, _ = TT.llm_logprobs(c, RSEED, "ref.", emb, grp.question, grp.resp, grp.lengths, "cuda")
    emb = emb.cpu().numpy()
    torch.cuda.empty_cache()
    return emb, lp_p, lp_r, {"oracle_vision_s": t1 - t0, "oracle_llm_s": time.time() - t1}


def _check(name, w, got, want, timing):
    emb, lp_p, lp_r, st = got
    oemb, olp_p, olp_r = want
    rec = _emb_stats(emb.astype(np.float64), oemb)
    for tag, a, b in (("policy", lp_p, olp_p), ("ref", lp_r, olp_r)):
        d = np.abs(a.astype(np.float64) - b)
        rec[f"lp_{tag}_max"], rec[f"lp_{tag}_mean"] = float(d.max()), float(d.mean())
    rec["scored"] = int(len(lp_p))
    rec.update(timing)
    _record(name, rec)
    print(name, rec)
    assert st["cache_misses"] == 1 and st["cache_hits"] == w.G - 1
    assert st["encoder_invocations"] == w.frames and st["pad_reads"] == 0
    assert rec["emb_rel_max"] <= EMB_REL and rec["emb_cos_min"] >= EMB_COS, rec
    for tag in ("policy", "ref"):
        assert rec[f"lp_{tag}_max"] <= LP_MAX and rec[f"lp_{tag}_mean"] <= LP_MEAN, rec


def test_c2_end_to_end_vs_oracle(gpu):
    """c2: 64 frames, SigLIP-shaped tower, 4-layer Qwen2.5-7B-shaped LLM, G = 8 —
    every embedding and every scored log-prob of both models; SP = 2 virtual
    ranks bit-identical to SP = 1."""
    w = E.workloads()["c2"]
    c = T.Cfg.from_any(w.cfg)
    pix = E.gen_video(1, w.frames, 3 * c.image_size ** 2)
    grp = E.make_group(w, seed=3)
    vid = E.video_id(1, w.frames)
    got1 = _engine(w, 1, pix, grp, vid)
    got2 = _engine(w, 2, pix, grp, vid)
    assert np.array_equal(got1[0], got2[0]), "SP=2 embeddings differ from SP=1"
    assert np.array_equal(got1[1], got2[1]) and np.array_equal(got1[2], got2[2]), \
        "SP=2 log-probs differ from SP=1"
    want_emb, want_p, want_r, timing = _oracle(w, pix, grp)
    _check("c2", w, got1, (want_emb, want_p, want_r), timing)


def test_c4_end_to_end_vs_oracle(gpu):
    """c4 (the bench workload): 512 frames x 256 tokens, 28-layer 7B-shaped LLM,
    G = 8, 131,109 prefix tokens — all 131,072 frame embeddings and all scored
    log-probs of both models."""
    w = E.workloads()["c4"]
    c = T.Cfg.from_any(w.cfg)
    pix = E.gen_video(1, w.frames, 3 * c.image_size ** 2)
    grp = E.make_group(w, seed=3)
    got = _engine(w, 1, pix, grp, E.video_id(1, w.frames))
    want_emb, want_p, want_r, timing = _oracle(w, pix, grp)
    _check("c4", w, got, (want_emb, want_p, want_r), timing)


def test_c2_generation_vs_oracle(gpu):
    """Rollout generation at c2 width (sample_rollout,
    policy.cpp:121-157): the old log-probs recorded while decoding G rows after
    the 16K-token prompt, against the float64 oracle's teacher-forced log-probs
    of the sampled tokens (its own tower and weights), at the §8c log-prob
    tolerance."""
    from oracle import transformer_torch as TT
    w = E.workloads()["c2"]
    c = T.Cfg.from_any(w.cfg)
    pix = E.gen_video(1, w.frames, 3 * c.image_size ** 2)
    q = np.arange(10, 10 + w.n_question, dtype=np.int32)
    eng = E.Engine(w.cfg, sp=1, vision_seed=VSEED, policy_seed=PSEED, ref_seed=RSEED, with_ref=False)
    eng.encode("v", pix)
    G, max_len = 8, 32
    tok, lens, olp = eng.generate("v", q, G, max_len, temperature=1.0, seed=5)
    eng.close()
    resp = np.zeros((G, max_len), dtype=np.int32)
    for g in range(G):
        resp[g, :lens[g]] = tok[g, :lens[g]]
    Wv = TT.vision_weights(c, VSEED, "cuda")
    emb = TT.vision_forward(c, Wv, pix, "cuda")
    del Wv
    want, _ = TT.llm_logprobs(c, PSEED, "policy.", emb, q, resp, lens, "cuda")
    torch.cuda.empty_cache()
    got = np.concatenate([olp[g, :lens[g]] for g in range(G)]).astype(np.float64)
    d = np.abs(got - want)
    rec = {"lp_max": float(d.max()), "lp_mean": float(d.mean()), "tokens": int(lens.sum())}
    _record("c2_generation", rec)
    print("c2 generation vs oracle", rec)
    assert d.max() <= LP_MAX and d.mean() <= LP_MEAN, rec
