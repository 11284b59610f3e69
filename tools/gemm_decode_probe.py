"""Decode-GEMM probe (dev tool): time the gate/up and down projections of a
decode step (M = G rows) in isolation with CUDA events, for M = 8 and 128 and
the skinny / default rings, against the pure weight-stream time."""
import json
import os
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch

from paper_2507_07966_b200 import ops


def t_ms(f, iters=50):
    for _ in range(3):
        f()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        f()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


for (N, K, epi, name) in [(37888, 3584, ops.EPI_SWIGLU_BF16, "gate/up swiglu"),
                          (3584, 18944, ops.EPI_STORE_F32, "down (fp32 out)")]:
    B = (torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16()
    for M in (8, 128):
        A = torch.randn(M, K, device="cuda").bfloat16()
        ws = torch.empty(ops.splitk_workspace_bytes(M), dtype=torch.uint8, device="cuda")
        for sk in ("1", "0"):
            os.environ["MRSP_GEMM_SKINNY"] = sk
            for split in (False, True):
                f = (lambda: ops.gemm(A, B, epi, splitk_ws=ws)) if split else (lambda: ops.gemm(A, B, epi))
                ms = t_ms(f)
                print(json.dumps({"gemm": name, "M": M, "N": N, "K": K, "skinny_env": sk, "splitk_ws": split,
                                  "us": round(ms * 1e3, 1), "weight_TBps": round(N * K * 2 / ms / 1e9, 2)}),
                      flush=True)
