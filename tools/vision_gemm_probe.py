"""Vision-tower GEMM probe (c4: 512 frames x 256 tokens) — dev tool, not the bench.

Times each SigLIP GEMM with its production epilogue and with a plain bf16 store,
next to cuBLAS, so the epilogue's share of a short-K tile is visible."""
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch

from paper_2507_07966_b200 import ops

M = 131072
# (name, N, K, production epilogue)
SHAPES = [("qkv", 6144, 1152, ops.EPI_BIAS_BF16), ("o", 1152, 2048, ops.EPI_RESID_F32),
          ("mlp_up", 4304, 1152, ops.EPI_BIAS_GELU_BF16), ("mlp_down", 1152, 4304, ops.EPI_RESID_F32)]


def timed(fn, iters=10):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main(only=None):
    for name, N, K, epi in SHAPES:
        if only and name not in only:
            continue
        A = torch.randn(M, K, device="cuda").bfloat16()
        B = (torch.randn(N, K, device="cuda") * 0.03).bfloat16()
        bias = torch.randn(N, device="cuda")
        resid = torch.zeros(M, N, device="cuda")
        out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        fl = 2 * M * N * K
        row = {"gemm": name, "M": M, "N": N, "K": K}
        if epi == ops.EPI_RESID_F32:
            f = lambda: ops.gemm(A, B, epi, bias=None, resid=resid)
        else:
            f = lambda: ops.gemm(A, B, epi, bias=bias, out=out)
        for tag, fn in [("prod", f), ("store", lambda: ops.gemm(A, B, ops.EPI_STORE_BF16, out=out)),
                        ("cublas", lambda: torch.mm(A, B.T))]:
            ms = timed(fn)
            row[tag + "_ms"] = round(ms, 3)
            row[tag + "_tflops"] = round(fl / ms / 1e9, 1)
        print(json.dumps(row), flush=True)
        del A, B, bias, resid, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main(sys.argv[1:])
