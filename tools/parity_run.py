#!/usr/bin/env python
"""Engine vs float64 oracle at a benchmarked configuration, end to end (dev
tool; the same check as tests/test_parity_configs_gpu.py, for the configs too
slow for the test suite — c3 takes minutes, c5 ~ an hour of float64 attention
over 262K tokens).

  MRSP_PARITY_OUT=profiles/r2_parity.jsonl python tools/parity_run.py c3 c5
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import test_parity_configs_gpu as P  # noqa: E402
from oracle import transformer as T  # noqa: E402
from paper_2507_07966_b200 import engine as E  # noqa: E402


def main():
    for name in sys.argv[1:] or ["c3"]:
        w = E.workloads()[name]
        c = T.Cfg.from_any(w.cfg)
        pix = E.gen_video(1, w.frames, 3 * c.image_size ** 2)
        grp = E.make_group(w, seed=3)
        got = P._engine(w, 1, pix, grp, E.video_id(1, w.frames))
        want_emb, want_p, want_r, timing = P._oracle(w, pix, grp)
        P._check(name, w, got, (want_emb, want_p, want_r), timing)


if __name__ == "__main__":
    main()
