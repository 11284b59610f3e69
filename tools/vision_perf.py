#!/usr/bin/env python
"""Stage-1 (SigLIP-shaped tower + projector) throughput probe (dev tool): one
cache-off encode of F frames through the engine, device time of the vision
class (engine profile), for the head-stride variants given on the command line
(MRSP_VISION_PAD=0: real head dim 72 with on-chip zero fill; 1: heads padded
to 128 in HBM), interleaved."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import transformer as T  # noqa: E402
from paper_2507_07966_b200 import engine as E  # noqa: E402


def main():
    frames = int(os.environ.get("FRAMES", "512"))
    pads = sys.argv[1:] or ["0", "1"]
    w = E.workloads()["c4"]
    d = w.cfg.as_dict()
    d["layers"] = 1
    cfg = E.ModelConfig(**d)
    c = T.Cfg.from_any(cfg)
    pix = E.gen_video(1, frames, 3 * c.image_size ** 2)
    flops = T.step_flops(c, frames, 0, [0], passes=0)["encode"]
    engines = {}
    for p in pads:
        os.environ["MRSP_VISION_PAD"] = p
        engines[p] = E.Engine(cfg, sp=1, with_ref=False)
    for rep in range(int(os.environ.get("REPS", "3"))):
        for p in pads:
            eng = engines[p]
            if os.environ.get("WARM", "1") == "1":
                eng.encode("warm", pix, use_cache=False)
            eng.profile(True)
            eng.encode("v", pix, use_cache=False)
            ms = eng.profile(False)["vision"][0]
            print(json.dumps({"pad": p, "rep": rep, "frames": frames, "vision_ms": round(ms, 2),
                              "tflops": round(flops / ms / 1e9, 1)}), flush=True)
    for eng in engines.values():
        eng.close()


if __name__ == "__main__":
    main()
