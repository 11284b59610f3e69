"""Rollout-generation throughput (dev tool): per-decode-step time from two
generate() calls of different length (prompt prefill cancels), against the
HBM roofline of a decode step (all LLM weights + the prompt K/V per step)."""
import sys, pathlib, json, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2507_07966_b200 import engine as E

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
G = int(sys.argv[2]) if len(sys.argv) > 2 else 8
w = E.workloads()[name]
c = w.cfg
eng = E.Engine(c, sp=1, with_ref=False)
S = c.image_size
pix = torch.from_numpy(E.gen_video(1, w.frames, 3 * S * S)).cuda()
eng.encode("v", pix)
q = np.arange(10, 10 + w.n_question, dtype=np.int32)
eng.generate("v", q, G, 4, seed=1)  # warm
t, prof = {}, {}
N1, N2 = 8, 136  # 128 decode steps apart: the prompt prefill (seconds) cancels
for n in (N1, N2):
    eng.profile(True)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    tok, lens, _ = eng.generate("v", q, G, n, seed=2)
    torch.cuda.synchronize(); t[n] = time.perf_counter() - t0
    prof[n] = eng.profile(False)
    assert (lens == n).all(), lens
# device time per decode step by class (prefill cancels in the difference)
per_step = {k: round((prof[N2][k][0] - prof[N1][k][0]) / (N2 - N1), 3) for k in prof[N2]}
step = (t[N2] - t[N1]) / (N2 - N1)
L, d, nq, nkv, mlp, V = c.layers, c.dim, c.n_q_heads, c.n_kv_heads, c.mlp, c.vocab
weights = 2 * (L * (d * (nq + 2 * nkv) * 128 + nq * 128 * d + 3 * d * mlp) + V * d)
Lp = w.frames * c.tokens_per_frame + w.n_question
kv = 2 * L * Lp * 2 * nkv * 128
peaks = json.load(open(pathlib.Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"))
ideal = (weights + kv) / (peaks["hbm_gbs"] * 1e9)
dev = sum(per_step.values()) / 1e3  # device busy time per decode step (s)
print(json.dumps({"workload": name, "G": G, "prompt_tokens": Lp, "prefill_plus_8_steps_s": round(t[N1], 3),
                  "device_step_ms": round(dev * 1e3, 3), "wall_step_ms": round(step * 1e3, 3),
                  "tokens_per_s_device": round(G / dev, 1), "hbm_bytes_per_step": weights + kv,
                  "hbm_roofline_step_ms": round(ideal * 1e3, 3),
                  "roofline_frac_device": round(ideal / dev, 3), "device_ms_per_step_by_class": per_step}),
      flush=True)
