"""GPU: rollout generation (sample_rollout, policy.cpp:121-157)
reusing the cached video embeddings and the prompt's K/V.

The sampled tokens are checked by teacher forcing: the log-probabilities
recorded while sampling (old_logprobs, temperature 1) must equal, within the
BF16/FP32 tolerance, (a) the engine's own prefill log-probs of the same tokens
(a different kernel path: full-sequence attention instead of decode attention
over the cached K/V) and (b) the numpy fp64 oracle's. Plus the reference's
sampling contract: EOS ends a row (and is its last token), PAD after it,
lengths, seed determinism, argument errors."""
import numpy as np
import pytest

from oracle import transformer as T
from paper_2507_07966_b200 import _lib, engine as E

pytestmark = pytest.mark.gpu

W1 = E.workloads()["c1"]
VSEED, PSEED, RSEED = 2, 3, 4
EOS, PAD = 1, 0


def _rows(tok, lens):
    G, max_len = tok.shape
    resp = np.zeros((G, max_len), dtype=np.int32)
    for g in range(G):
        resp[g, :lens[g]] = tok[g, :lens[g]]
    return resp


@pytest.fixture(scope="module")
def gen():
    c = T.Cfg.from_any(W1.cfg)
    pix = E.gen_video(1, W1.frames, 3 * c.image_size ** 2)
    q = np.array([10, 11, 12], dtype=np.int32)
    eng = E.Engine(W1.cfg, sp=1, vision_seed=VSEED, policy_seed=PSEED, ref_seed=RSEED)
    eng.encode("v", pix)
    G, max_len = 16, 24
    tok, lens, olp = eng.generate("v", q, G, max_len, temperature=1.0, seed=7)
    yield dict(eng=eng, pix=pix, q=q, tok=tok, lens=lens, olp=olp, c=c)
    eng.close()


def test_generation_contract(gpu, gen):
    tok, lens, olp = gen["tok"], gen["lens"], gen["olp"]
    G, max_len = tok.shape
    assert ((lens >= 1) & (lens <= max_len)).all()
    for g in range(G):
        n = lens[g]
        body = tok[g, :n]
        assert ((body >= 0) & (body < W1.cfg.vocab)).all()
        assert (body[:-1] != EOS).all(), "EOS must end the row"
        assert n == max_len or body[-1] == EOS
        assert (tok[g, n:] == PAD).all() and (olp[g, :n] <= 0).all()
    assert (lens < max_len).any() or (tok == EOS).sum() == 0  # V = 32: some rows end early


def test_old_logprobs_match_prefill_and_oracle(gpu, gen):
    eng, q, tok, lens, olp, c = gen["eng"], gen["q"], gen["tok"], gen["lens"], gen["olp"], gen["c"]
    resp = _rows(tok, lens)
    grp = E.Group(q, resp, lens.astype(np.int32))
    want_engine = eng.prefill_logprobs("v", grp, 0)
    got = np.concatenate([olp[g, :lens[g]] for g in range(len(lens))])
    d = np.abs(got - want_engine)
    assert d.max() <= 5e-2 and d.mean() <= 5e-3, ("vs engine prefill", d.max(), d.mean())
    emb = T.vision_forward(c, T.vision_weights(c, VSEED), gen["pix"])
    want_oracle, _ = T.llm_logprobs(c, T.llm_weights(c, PSEED, "policy."), emb, q, resp, lens)
    d = np.abs(got - want_oracle)
    assert d.max() <= 5e-2 and d.mean() <= 5e-3, ("vs oracle", d.max(), d.mean())


def test_seed_determinism_and_errors(gpu, gen):
    eng, q = gen["eng"], gen["q"]
    a = eng.generate("v", q, 4, 10, temperature=0.7, seed=123)
    b = eng.generate("v", q, 4, 10, temperature=0.7, seed=123)
    c = eng.generate("v", q, 4, 10, temperature=0.7, seed=124)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    assert not np.array_equal(a[0], c[0])
    with pytest.raises(_lib.InvalidArgument):
        eng.generate("v", q, 4, 10, temperature=0.0)  # sample_rollout: temperature must be > 0
    with pytest.raises(_lib.InvalidArgument):
        eng.generate("v", q, 4, 0)  # max_len must be >= 1


@pytest.mark.parametrize("env", [{"MRSP_DECODE_CC": "0"}, {"MRSP_DECODE_CC": "1"},
                                 {"MRSP_DECODE_RING": "6"},
                                 {"MRSP_DECODE_RING": "6", "MRSP_DECODE_STREAMS": "1"}],
                         ids=["tc-ring2", "cuda-cores", "tc-ring6-2streams", "tc-ring6-1stream"])
def test_decode_kernels_agree(gpu, gen, env, monkeypatch):
    """Every decode-attention variant (tcgen05 with two CTAs per SM; tcgen05 with
    one CTA per SM and two or one KV streams; CUDA cores) gives old log-probs that
    match the engine's prefill of the sampled tokens. At c1 (515 prompt keys,
    512-key chunks) the second chunk's second stream has no tile (empty partial)."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    cc = env.get("MRSP_DECODE_CC", "0")
    eng, q = gen["eng"], gen["q"]
    tok, lens, olp = eng.generate("v", q, 8, 16, temperature=0.8, seed=99)
    grp = E.Group(q, _rows(tok, lens), lens.astype(np.int32))
    want = eng.prefill_logprobs("v", grp, 0)
    got = np.concatenate([olp[g, :lens[g]] for g in range(len(lens))])
    d = np.abs(got - want)
    assert d.max() <= 5e-2 and d.mean() <= 5e-3, (cc, d.max(), d.mean())


@pytest.mark.parametrize("ring", ["", "6"], ids=["default", "ring6-2streams"])
def test_graph_replay_matches_eager(gpu, gen, ring, monkeypatch):
    """Steps t >= 1 replay one captured CUDA graph whose attention grid is sized
    for t = max_len - 1 (chunks past the live row keys are empty): tokens,
    lengths and old log-probs are bit-identical to launching every step eagerly.
    G x max_len = 640 row keys, so early steps run with an empty row chunk."""
    eng, q = gen["eng"], gen["q"]
    if ring:
        monkeypatch.setenv("MRSP_DECODE_RING", ring)
    monkeypatch.setenv("MRSP_DECODE_GRAPH", "0")
    eager = eng.generate("v", q, 16, 40, temperature=0.9, seed=5)
    monkeypatch.setenv("MRSP_DECODE_GRAPH", "1")
    graph = eng.generate("v", q, 16, 40, temperature=0.9, seed=5)
    for x, y in zip(eager, graph):
        assert np.array_equal(x, y)


def test_decode_fusions(gpu, monkeypatch):
    """c2 shapes (d 3584, K split over the SMs). The fused decode kernels —
    embedding + first RMSNorm, QKV split-K reduction + RoPE + row-cache append,
    residual split-K reduction + the next RMSNorm (one 4-CTA cluster per row) —
    and the separate kernels (MRSP_DECODE_FUSE=0) each give graph replays
    bit-identical to eager steps, and old log-probs that match the engine's
    prefill of the sampled tokens."""
    w = E.workloads()["c2"]
    c = T.Cfg.from_any(w.cfg)
    eng = E.Engine(w.cfg, sp=1, with_ref=False)
    try:
        eng.encode("v", E.gen_video(1, w.frames, 3 * c.image_size ** 2))
        q = np.arange(10, 10 + w.n_question, dtype=np.int32)
        for fuse in ("0", "1"):
            monkeypatch.setenv("MRSP_DECODE_FUSE", fuse)
            out = {}
            for graph in ("0", "1"):
                monkeypatch.setenv("MRSP_DECODE_GRAPH", graph)
                out[graph] = eng.generate("v", q, 4, 6, temperature=1.0, seed=11)
            for x, y in zip(out["0"], out["1"]):
                assert np.array_equal(x, y), fuse
            tok, lens, olp = out["1"]
            grp = E.Group(q, _rows(tok, lens), lens.astype(np.int32))
            want = eng.prefill_logprobs("v", grp, 0)
            got = np.concatenate([olp[g, :lens[g]] for g in range(len(lens))])
            d = np.abs(got - want)
            assert d.max() <= 5e-2 and d.mean() <= 5e-3, (fuse, d.max(), d.mean())
    finally:
        eng.close()


def test_generation_edges(gpu, gen):
    """One rollout row (G = 1) and the largest group a decode-attention Q tile
    holds (G x q_per_kv <= 64) sample under the same contract; one row more is
    an invalid argument (generate's own limit, not the reference's)."""
    eng, q, c = gen["eng"], gen["q"], gen["c"]
    qpk = c.n_q_heads // c.n_kv_heads
    g_max = 64 // qpk
    for G in (1, g_max):
        tok, lens, olp = eng.generate("v", q, G, 9, temperature=1.0, seed=3)
        assert tok.shape == (G, 9) and ((lens >= 1) & (lens <= 9)).all()
        grp = E.Group(q, _rows(tok, lens), lens.astype(np.int32))
        want = eng.prefill_logprobs("v", grp, 0)
        got = np.concatenate([olp[g, :lens[g]] for g in range(G)])
        d = np.abs(got - want)
        assert d.max() <= 5e-2 and d.mean() <= 5e-3, (G, d.max(), d.mean())
    with pytest.raises(_lib.InvalidArgument):
        eng.generate("v", q, g_max + 1, 4)


@pytest.mark.parametrize("sp", [2, 4, 8])
def test_generation_sp_bit_exact(gpu, gen, sp):
    """Generation inside an SP engine (grpo.cpp:376-386): the prompt prefill
    runs sequence-parallel over `sp` virtual ranks (at SP 8 > n_kv the kv
    heads are shared by query-row split ranks), the prompt K/V of every kv head
    is gathered from the ranks' head shards, and the sampled tokens, lengths
    and old log-probs are bit-identical to SP = 1."""
    eng1, q = gen["eng"], gen["q"]
    want = eng1.generate("v", q, 8, 20, temperature=1.0, seed=21)
    eng = E.Engine(W1.cfg, sp=sp, vision_seed=VSEED, policy_seed=PSEED, ref_seed=RSEED)
    try:
        eng.encode("v", gen["pix"])
        got = eng.generate("v", q, 8, 20, temperature=1.0, seed=21)
    finally:
        eng.close()
    for x, y in zip(want, got):
        assert np.array_equal(x, y), sp
