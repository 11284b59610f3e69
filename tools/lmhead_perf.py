#!/usr/bin/env python
"""Fused dual LM head throughput (CUDA events, dev tool): mrsp_op_lmhead_dual at
the c2-c5 scored-token count (M = 6551, V = 152064, K = 3584), TFLOP/s against
the 2 x 2 M V K algorithmic FLOPs of the two vocabulary projections."""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_07966_b200 import _lib  # noqa: E402


def vp(t):
    return ctypes.c_void_p(t.data_ptr())


def main(M=6551, V=152064, K=3584, iters=20):
    Xp = torch.randn(M, K, device="cuda").bfloat16()
    Xr = torch.randn(M, K, device="cuda").bfloat16()
    Wp = (torch.randn(V, K, device="cuda") / K ** 0.5).bfloat16()
    Wr = (torch.randn(V, K, device="cuda") / K ** 0.5).bfloat16()
    tgt = torch.randint(0, V, (M,), device="cuda", dtype=torch.int32)
    out = [torch.empty(M, device="cuda") for _ in range(3)]
    wsb = _lib.lib().mrsp_lmhead_dual_workspace_bytes(M, V)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream

    def call():
        _lib.check(_lib.lib().mrsp_op_lmhead_dual(vp(Xp), vp(Wp), vp(Xr), vp(Wr), M, V, K, vp(tgt),
                                                  vp(out[0]), vp(out[1]), vp(out[2]), vp(ws), wsb,
                                                  ctypes.c_void_p(stream)))
    for _ in range(3):
        call()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        call()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / iters
    print(json.dumps({"M": M, "V": V, "K": K, "ms": round(ms, 3),
                      "tflops": round(4 * M * V * K / ms / 1e9, 1)}))


if __name__ == "__main__":
    main(*[int(x) for x in sys.argv[1:]])
