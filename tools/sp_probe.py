#!/usr/bin/env python
"""SP-invariance probe (GPU): c1 through the engine at SP = 1, 2, 4, 6, 8
virtual ranks; prints, per SP degree, how many embedding / log-prob values
differ from SP = 1 and by how much (0 everywhere = bit-identical)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_07966_b200 import engine as E  # noqa: E402


def run(w, sp, pix, grp):
    eng = E.Engine(w.cfg, sp=sp, vision_seed=2, policy_seed=3, ref_seed=4)
    eng.encode("v", pix)
    emb = eng.embeddings("v")
    lp_p = eng.prefill_logprobs("v", grp, 0)
    lp_r = eng.prefill_logprobs("v", grp, 1)
    eng.close()
    return emb, lp_p, lp_r


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c1"
    sps = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [2, 4, 6, 8]
    w = E.workloads()[name]
    pix = E.gen_video(1, w.frames, 3 * w.cfg.image_size ** 2)
    grp = E.make_group(w, seed=3)
    base = run(w, 1, pix, grp)
    for sp in sps:
        got = run(w, sp, pix, grp)
        rec = {"workload": name, "sp": sp}
        for tag, a, b in zip(("emb", "lp_policy", "lp_ref"), got, base):
            rec[tag + "_ndiff"] = int((a != b).sum())
            rec[tag + "_maxdiff"] = float(np.abs(a - b).max())
            if tag != "emb" and rec[tag + "_ndiff"]:
                rec[tag + "_first"] = int(np.argmax(a != b))
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
