"""Run one MR-SP step for a workload on 1 GPU (SP=1) and print per-class device time."""
import sys, pathlib, json, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_2507_07966_b200 import engine as E
from oracle import transformer as T

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w = E.workloads()[name]
t0 = time.time()
eng = E.Engine(w.cfg, sp=1)
print("init s", round(time.time() - t0, 1), flush=True)
S = w.cfg.image_size
pix = torch.from_numpy(E.gen_video(1, w.frames, 3 * S * S)).cuda()
grp = E.make_group(w)
fl = T.step_flops(T.Cfg.from_any(w.cfg), w.frames, w.n_question, grp.lengths)
eng.step("warm", pix, grp)
for i in range(steps):
    eng.profile(True)
    torch.cuda.synchronize()
    t = time.time()
    eng.step(f"s{i}", pix, grp)
    torch.cuda.synchronize()
    dt = time.time() - t
    prof = eng.profile(False)
    print(json.dumps({"workload": name, "step_s": round(dt, 3), "tokens": fl["tokens"],
                      "tok_per_s": round(fl["tokens"] / dt, 1), "tflops": round(fl["step"] / dt / 1e12, 1),
                      "prof_ms": {k: [round(v[0], 1), v[1]] for k, v in prof.items()},
                      "attn_tflops": round(2 * (fl["attn_prefix"] + fl["attn_resp"]) / (prof["llm_attention"][0] / 1e3) / 1e12, 1),
                      "gemm_tflops": round(2 * fl["linear"] / (prof["llm_gemm"][0] / 1e3) / 1e12, 1),
                      "vision_tflops": round(fl["encode"] / (prof["vision"][0] / 1e3) / 1e12, 1)}), flush=True)
