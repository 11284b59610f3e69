"""Determinism check of the attention kernel (bitwise reruns) — dev tool."""
import sys, pathlib, math, os
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_2507_07966_b200 import ops
L, nq, nkv, Lp, Lmax = 4096 + 8 * 300, 7, 1, 4096, 300
g = torch.Generator(device="cuda").manual_seed(0)
qkv = torch.randn(L, (nq + 2 * nkv) * 128, device="cuda", generator=g).bfloat16()
def run(poly):
    os.environ["MRSP_ATTN_POLY"] = poly
    o = ops.attention(qkv, 0, qkv, nq * 128, qkv, (nq + nkv) * 128, L, nq, nq // nkv, 1 / math.sqrt(128), 0, Lp, Lmax, 0)
    torch.cuda.synchronize(); return o.float()
for poly in ("0", "8"):
    ref = run(poly)
    nbad = []
    for rep in range(10):
        d = (run(poly) - ref).abs().view(L, nq, 128).amax(-1)
        nbad.append(int((d > 0).sum().item()))
    print(f"poly {poly}: rows differing from run 0 over 10 reruns: {nbad}", flush=True)
