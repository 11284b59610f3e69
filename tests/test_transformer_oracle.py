"""CPU: the transformer-shaped oracle's own invariants (layout, mask, init,
FLOP table against BASELINE.md §4)."""
import numpy as np

from oracle import transformer as T
from paper_2507_07966_b200 import engine as E


def test_bf16_round_matches_torch():
    import torch
    x = np.random.default_rng(0).standard_normal(10000).astype(np.float32) * 10
    assert np.array_equal(T.bf16_round(x), torch.from_numpy(x).bfloat16().float().numpy())


def test_init_is_deterministic_and_scaled():
    a = T.init_bf16((64, 128), 3, "policy.0.wqkv", T.wscale(128))
    b = T.init_bf16((64, 128), 3, "policy.0.wqkv", T.wscale(128))
    c = T.init_bf16((64, 128), 4, "policy.0.wqkv", T.wscale(128))
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    assert abs(a.std() - 1 / np.sqrt(128)) < 0.01
    n = T.init_f32((1000,), 1, "x.norm", T.K_NORM, 1.0)
    assert 0.9 <= n.min() and n.max() <= 1.1


def test_pack_layout_matches_pad_batch_semantics():
    resp = np.array([[5, 6, 7, 0], [8, 0, 0, 0], [9, 10, 11, 12]], dtype=np.int32)
    lengths = np.array([3, 1, 4])
    tok, pos, pad, Lp, L = T.pack(4, [20, 21], resp, lengths)
    assert Lp == 6 and L == 6 + 12
    assert tok[:4].tolist() == [-1] * 4 and tok[4:6].tolist() == [20, 21]
    assert tok[6:10].tolist() == [1, 5, 6, 0]      # EOS, y0, y1, PAD
    assert tok[10:14].tolist() == [1, 0, 0, 0]
    assert tok[14:18].tolist() == [1, 9, 10, 11]
    assert pad.tolist() == [0] * 6 + [0, 0, 0, 1] + [0, 1, 1, 1] + [0, 0, 0, 0]
    assert pos[6:10].tolist() == [6, 7, 8, 9] and pos[14:18].tolist() == [6, 7, 8, 9]


def test_mask_rows_see_prefix_and_themselves():
    m = T.mrsp_mask(10, 4, 3)
    assert m[5, :5].tolist() == [1, 1, 1, 1, 1]
    assert not m[7, 4] and not m[7, 5] and not m[7, 6] and m[7, 7] and m[7, 3]
    assert not m[2, 3] and m[3, 3]


def test_flop_table_matches_baseline_md():
    """c4 step ≈ 1.13e16 FLOP, c2 ≈ 1.40e14 (with Σℓ=6160)."""
    w = E.workloads()
    lens = [770] * 8  # Σℓ = 6160 as in the survey's table
    c4 = T.step_flops(T.Cfg.from_any(w["c4"].cfg), 512, 37, lens)
    assert abs(c4["step"] / 1.13e16 - 1) < 0.02, c4["step"]
    assert c4["Lp"] == 131109
    c2 = T.step_flops(T.Cfg.from_any(w["c2"].cfg), 64, 37, lens)
    assert abs(c2["step"] / 1.40e14 - 1) < 0.03, c2["step"]
    assert abs(c4["encode"] / 512 / 227.7e9 - 1) < 0.01


def test_c1_oracle_runs_end_to_end():
    w = E.workloads()["c1"]
    c = T.Cfg.from_any(w.cfg)
    pix = E.gen_video(1, w.frames, 3 * c.image_size ** 2)
    grp = E.make_group(w)
    emb = T.vision_forward(c, T.vision_weights(c, 2), pix)
    assert emb.shape == (w.frames * c.T, c.dim) and np.isfinite(emb).all()
    lp, lse = T.llm_logprobs(c, T.llm_weights(c, 3, "policy."), emb, grp.question, grp.resp,
                             grp.lengths)
    assert lp.shape == (grp.scored,) and (lp < 0).all() and np.isfinite(lse).all()
