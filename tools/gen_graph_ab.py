"""Decode-step A/B (dev tool): every step launched eagerly vs one CUDA graph
replay per step (MRSP_DECODE_GRAPH), with and without programmatic dependent
launch inside the graph (MRSP_DECODE_PDL). Wall time per decode step from two
generate() calls of different length (the prompt prefill cancels), profiling
off; then the device time per step from the engine's event classes.

  python tools/gen_graph_ab.py [workload ...]     # default: c2 c4
"""
import json
import os
import pathlib
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2507_07966_b200 import engine as E

N1, N2 = 8, 72


def per_step(eng, q, G, mode, profile):
    os.environ["MRSP_DECODE_GRAPH"], os.environ["MRSP_DECODE_PDL"] = mode
    wall, dev = {}, {}
    for n in (N1, N2):
        if profile:
            eng.profile(True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tok, lens, _ = eng.generate("v", q, G, n, temperature=1.0, seed=2)
        torch.cuda.synchronize()
        wall[n] = time.perf_counter() - t0
        if profile:
            dev[n] = sum(v[0] for v in eng.profile(False).values())
        assert (lens == n).all(), lens
    out = {"wall_step_ms": round((wall[N2] - wall[N1]) / (N2 - N1) * 1e3, 3)}
    if profile:
        out["device_step_ms"] = round((dev[N2] - dev[N1]) / (N2 - N1), 3)
    return out


def main(names):
    peaks = json.load(open(pathlib.Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"))
    for name in names:
        w = E.workloads()[name]
        c = w.cfg
        G = 8
        eng = E.Engine(c, sp=1, with_ref=False)
        S = c.image_size
        pix = torch.from_numpy(E.gen_video(1, w.frames, 3 * S * S)).cuda()
        eng.encode("v", pix)
        q = np.arange(10, 10 + w.n_question, dtype=np.int32)
        eng.generate("v", q, G, 4, seed=1)  # warm
        L, d, nq, nkv, mlp, V = c.layers, c.dim, c.n_q_heads, c.n_kv_heads, c.mlp, c.vocab
        weights = 2 * (L * (d * (nq + 2 * nkv) * 128 + nq * 128 * d + 3 * d * mlp) + V * d)
        Lp = w.frames * c.tokens_per_frame + w.n_question
        bound_ms = (weights + 2 * L * Lp * 2 * nkv * 128) / (peaks["hbm_gbs"] * 1e9) * 1e3
        for rnd in range(2):
            modes = (("0", "0"), ("1", "0"), ("1", "1"))
            if os.environ.get("GEN_AB_GRAPH_ONLY"):
                modes = (("1", "0"),)
            for mode in modes:
                r = per_step(eng, q, G, mode, profile=False)
                r.update(per_step(eng, q, G, mode, profile=True))
                r.update({"workload": name, "G": G, "prompt_tokens": Lp, "graph": mode[0] == "1", "pdl": mode[1] == "1",
                          "streams": os.environ.get("MRSP_DECODE_STREAMS", "default"),
                          "fuse": os.environ.get("MRSP_DECODE_FUSE", "default"),
                          "round": rnd, "hbm_bound_step_ms": round(bound_ms, 3),
                          "hbm_frac_wall": round(bound_ms / r["wall_step_ms"], 3)})
                print(json.dumps(r), flush=True)
        eng.close()


if __name__ == "__main__":
    main(sys.argv[1:] or ["c2", "c4"])
