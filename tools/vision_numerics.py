#!/usr/bin/env python
"""Numerics probe for the SigLIP-shaped tower at production width (GPU).

Compares the engine's projector embeddings (1-2 frames) with the float64 twin
of the oracle (oracle/transformer_torch.py) in several arithmetic variants, to
separate the error every bf16-storing implementation has (oracle bf16 vs exact)
from what the engine's kernels add (bf16 P in attention, SFU tanh in GELU):

  exact       float64, no storage rounding
  bf16        the oracle: bf16 activations / fp32 residual (the parity target)
  bf16+P      + attention probabilities rounded to bf16 before P.V (flash style)

  python tools/vision_numerics.py [--lib path/to/libmrsp_b200.so] [--frames 2]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import transformer as T, transformer_torch as TT  # noqa: E402
from paper_2507_07966_b200 import _lib  # noqa: E402


def stats(a, b):
    rel = np.linalg.norm(a - b, axis=1) / np.linalg.norm(b, axis=1)
    cos = (a * b).sum(1) / (np.linalg.norm(a, axis=1) * np.linalg.norm(b, axis=1))
    return {"rel_max": float(rel.max()), "rel_mean": float(rel.mean()), "cos_min": float(cos.min())}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=None)
    ap.add_argument("--frames", type=int, default=2)
    ap.add_argument("--tag", default="default")
    a = ap.parse_args()
    if a.lib:
        _lib.LIB_PATH = type(_lib.LIB_PATH)(os.path.abspath(a.lib))
    from paper_2507_07966_b200 import engine as E
    w4 = E.workloads()["c4"]
    d = w4.cfg.as_dict()
    d["layers"] = 1
    cfg = E.ModelConfig(**d)
    c = T.Cfg.from_any(cfg)
    pix = E.gen_video(5, a.frames, 3 * c.image_size ** 2)
    eng = E.Engine(cfg, sp=1, vision_seed=2, policy_seed=3, ref_seed=4, with_ref=False)
    eng.encode("v", pix)
    emb = eng.embeddings("v").astype(np.float64)
    eng.close()
    dev = "cuda"
    W = TT.vision_weights(c, 2, dev)
    out = {}
    ref_bf16 = TT.vision_forward(c, W, pix, dev).cpu().numpy()
    b_, s_ = TT._b, TT._s
    TT._b = TT._s = lambda x: x
    ref_exact = TT.vision_forward(c, W, pix, dev).cpu().numpy()
    TT._b, TT._s = b_, s_
    fa = TT.frame_attention

    def pb16(q, k, v, scale):
        s = (q @ k.transpose(-1, -2)) * scale
        p = torch.exp(s - s.amax(-1, keepdim=True))
        return (p.to(torch.float32).to(torch.bfloat16).to(torch.float64) @ v) / p.sum(-1, keepdim=True)
    TT.frame_attention = pb16
    ref_p = TT.vision_forward(c, W, pix, dev).cpu().numpy()
    TT.frame_attention = fa
    out["oracle_bf16_vs_exact"] = stats(ref_bf16, ref_exact)
    out["oracle_bf16P_vs_exact"] = stats(ref_p, ref_exact)
    out["engine_vs_oracle_bf16"] = stats(emb, ref_bf16)
    out["engine_vs_exact"] = stats(emb, ref_exact)
    out["engine_vs_oracle_bf16P"] = stats(emb, ref_p)
    print(json.dumps({"tag": a.tag, "lib": a.lib or "default", **out}))


if __name__ == "__main__":
    main()
