"""Attention throughput probe (CUDA events) — dev tool.

  python tools/attn_perf.py [poly[:split] ...]   # sweep MRSP_ATTN_POLY / MRSP_ATTN_SPLIT
  (variants interleaved per shape, repeated `MRSP_PERF_REPS` times: clocks drift
  under the power cap)
"""
import sys, pathlib, json, math, os
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_2507_07966_b200 import ops

def bench(L, nq, nkv, Lp=None, Lmax=0, iters=5):
    qkv = torch.randn(L, (nq + 2 * nkv) * 128, device="cuda").bfloat16()
    out = torch.empty(L, nq * 128, device="cuda", dtype=torch.bfloat16)
    f = lambda: ops.attention(qkv, 0, qkv, nq*128, qkv, (nq+nkv)*128, L, nq, nq//nkv, 1/math.sqrt(128), 0, Lp, Lmax, 0, out=out)
    for _ in range(2): f()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); s.record()
    for _ in range(iters): f()
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / iters
    Lp_ = L if Lp is None else Lp
    G = (L - Lp_) // Lmax if Lmax else 0
    flops = 2 * 2 * 128 * nq * (Lp_ * Lp_ / 2 + G * (Lmax * Lp_ + Lmax * Lmax / 2))
    return dict(L=L, nq=nq, nkv=nkv, Lp=Lp_, Lmax=Lmax, ms=round(ms, 3), tflops=round(flops / ms / 1e9, 1))

if __name__ == "__main__":
    variants = sys.argv[1:] or [os.environ.get("MRSP_ATTN_POLY", "0")]
    reps = int(os.environ.get("MRSP_PERF_REPS", "1"))
    shapes = [(16384, 28, 4), (32768, 28, 4), (16421 + 8 * 1024, 28, 4, 16421, 1024),
              (131109 + 8 * 1011, 28, 4, 131109, 1011)]
    for args in shapes:
        for rep in range(reps):
            for v in variants:
                poly, _, split = v.partition(":")
                os.environ["MRSP_ATTN_POLY"] = poly or "0"
                os.environ["MRSP_ATTN_SPLIT"] = split or "1"
                r = bench(*args, iters=2 if args[0] > 100000 else 5)
                r["poly"], r["split"], r["rep"] = poly or "0", split or "1", rep
                print(json.dumps(r), flush=True)
