#!/usr/bin/env python
"""GRPO backward throughput probe (dev tool): mrsp_engine_grpo_backward on one
workload (env WORKLOAD, default c2) at SP = 1 — the reference pass, the policy
pass keeping layer inputs, the dual LM head, then the backward of every layer
(recompute + dgrad / wgrad GEMMs + tcgen05 attention backward). Prints wall
time per call, the engine's per-class device times and the attention-backward
kernels' algorithmic TFLOP/s (2.5x the forward attention FLOPs: S, dP, dQ, dK,
dV; the two-kernel design recomputes S and dP once more)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import transformer as T  # noqa: E402
from paper_2507_07966_b200 import engine as E  # noqa: E402


def main():
    wname = os.environ.get("WORKLOAD", "c2")
    reps = int(os.environ.get("REPS", "3"))
    w = E.workloads()[wname]
    c = T.Cfg.from_any(w.cfg)
    eng = E.Engine(w.cfg, sp=1)
    pix = E.gen_video(1, w.frames, 3 * c.image_size ** 2)
    grp = E.make_group(w, seed=3)
    vid = E.video_id(1, w.frames)
    eng.encode(vid, pix)
    lp = eng.prefill_logprobs(vid, grp, 0)
    rng = np.random.default_rng(0)
    old = lp - rng.normal(0, 0.1, size=lp.shape).astype(np.float32)
    adv = rng.normal(0, 1, size=w.G).astype(np.float32)
    fl = T.step_flops(c, w.frames, len(grp.question), list(grp.lengths), passes=1)
    L = w.frames * c.T + len(grp.question) + grp.resp.size
    eng.grpo_backward(vid, grp, old, adv)  # warm-up (allocations)
    for r in range(reps):
        eng.profile(True)
        t0 = time.perf_counter()
        st, _ = eng.grpo_backward(vid, grp, old, adv)
        wall = time.perf_counter() - t0
        prof = eng.profile(False)
        attn_fwd = fl["attn_prefix"] + fl["attn_resp"]  # one pass, all layers
        print(json.dumps({
            "workload": wname, "rep": r, "wall_ms": round(wall * 1e3, 1),
            "tokens": int(fl["tokens"]), "packed_tokens": L,
            "tokens_per_s": round(fl["tokens"] / wall, 1),
            "objective": st["objective"],
            "class_ms": {k: round(v[0], 2) for k, v in prof.items()},
            "attn_fwd_flops_per_pass": attn_fwd,
            "linear_flops_per_pass": fl["linear"],
        }), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
