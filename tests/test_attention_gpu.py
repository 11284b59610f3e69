"""GPU: tcgen05 flash attention (csrc/attention.cu) vs a plain PyTorch fp32
reference with the MR-SP shared-prefix mask, GQA, and the vision block mask."""
import math

import pytest
import torch

from paper_2507_07966_b200 import ops

pytestmark = pytest.mark.gpu


def ref_attn(qkv, L, nq, nkv, scale, mask):
    hd = 128
    q = qkv[:, : nq * hd].float().view(L, nq, hd).transpose(0, 1)
    k = qkv[:, nq * hd:(nq + nkv) * hd].float().view(L, nkv, hd).transpose(0, 1)
    v = qkv[:, (nq + nkv) * hd:(nq + 2 * nkv) * hd].float().view(L, nkv, hd).transpose(0, 1)
    rep = nq // nkv
    k = k.repeat_interleave(rep, 0)
    v = v.repeat_interleave(rep, 0)
    s = (q @ k.transpose(1, 2)) * scale
    s = s.masked_fill(~mask[None], float("-inf"))
    p = torch.softmax(s, -1)
    return (p @ v).transpose(0, 1).reshape(L, nq * hd)


def run(L, nq, nkv, mode, Lp=None, Lmax=0, blk=0, amp=1.0, hd_real=128, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    qkv = torch.randn(L, (nq + 2 * nkv) * 128, device="cuda", generator=g)
    if hd_real < 128:  # zero-padded heads (vision tower, hd 72)
        qkv.view(L, nq + 2 * nkv, 128)[:, :, hd_real:] = 0
    qkv[:, : nq * 128] *= amp
    qkv = qkv.bfloat16()
    scale = 1.0 / math.sqrt(hd_real)
    out = ops.attention(qkv, 0, qkv, nq * 128, qkv, (nq + nkv) * 128, L, nq, nq // nkv, scale,
                        mode, Lp, Lmax, blk)
    mask = ops.attention_mask(L, mode, Lp, Lmax, blk, device="cuda")
    want = ref_attn(qkv, L, nq, nkv, scale, mask)
    torch.cuda.synchronize()
    err = (out.float() - want).abs().max().item()
    rel = ((out.float() - want).norm() / want.norm()).item()
    return err, rel


def test_causal_prefix_gqa_small(gpu):
    err, rel = run(L=300 + 4 * 50, nq=4, nkv=2, mode=ops.ATTN_CAUSAL_PREFIX, Lp=300, Lmax=50)
    assert rel < 1e-2 and err < 5e-2, (err, rel)


def test_c1_shape(gpu):
    # c1: Lp 515 (8 frames x 64 + 3 question tokens), G 4 rows of Lmax 12
    err, rel = run(L=515 + 4 * 12, nq=4, nkv=2, mode=ops.ATTN_CAUSAL_PREFIX, Lp=515, Lmax=12)
    assert rel < 1e-2 and err < 5e-2, (err, rel)


def test_pure_causal_unaligned(gpu):
    err, rel = run(L=1000, nq=2, nkv=1, mode=ops.ATTN_CAUSAL_PREFIX)
    assert rel < 1e-2 and err < 5e-2, (err, rel)


def test_large_scores_trigger_rescale(gpu):
    err, rel = run(L=777, nq=2, nkv=2, mode=ops.ATTN_CAUSAL_PREFIX, Lp=500, Lmax=70, amp=6.0)
    assert rel < 2e-2, (err, rel)


def test_vision_block_diag_hd72(gpu):
    err, rel = run(L=1024, nq=2, nkv=2, mode=ops.ATTN_BLOCK_DIAG, blk=256, hd_real=72)
    assert rel < 1e-2 and err < 5e-2, (err, rel)


def test_qwen_gqa_7_to_1_long(gpu):
    err, rel = run(L=4096 + 8 * 300, nq=7, nkv=1, mode=ops.ATTN_CAUSAL_PREFIX, Lp=4096, Lmax=300)
    assert rel < 1e-2 and err < 5e-2, (err, rel)


@pytest.mark.parametrize("poly", ["0", "4", "8", "12", "16"])
def test_exp2_share_variants(gpu, poly, monkeypatch):
    # every FMA-pipe exp2 share (MRSP_ATTN_POLY) against the fp32 reference,
    # including masked tiles, a forced O rescale and the vision block mask
    monkeypatch.setenv("MRSP_ATTN_POLY", poly)
    err, rel = run(L=600 + 4 * 90, nq=4, nkv=2, mode=ops.ATTN_CAUSAL_PREFIX, Lp=600, Lmax=90)
    assert rel < 1e-2 and err < 5e-2, (poly, err, rel)
    err, rel = run(L=777, nq=2, nkv=2, mode=ops.ATTN_CAUSAL_PREFIX, Lp=500, Lmax=70, amp=6.0)
    assert rel < 2e-2, (poly, err, rel)
    err, rel = run(L=1024, nq=2, nkv=2, mode=ops.ATTN_BLOCK_DIAG, blk=256, hd_real=72)
    assert rel < 1e-2 and err < 5e-2, (poly, err, rel)
