"""Diff attention kernel generations (MRSP_ATTN_IMPL) row by row — dev tool."""
import sys, pathlib, math, os
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_2507_07966_b200 import ops

def run(L, nq, nkv, Lp, Lmax, impl, poly="8", seed=0):
    os.environ["MRSP_ATTN_IMPL"] = impl
    os.environ["MRSP_ATTN_POLY"] = poly
    g = torch.Generator(device="cuda").manual_seed(seed)
    qkv = torch.randn(L, (nq + 2 * nkv) * 128, device="cuda", generator=g).bfloat16()
    out = ops.attention(qkv, 0, qkv, nq * 128, qkv, (nq + nkv) * 128, L, nq, nq // nkv,
                        1 / math.sqrt(128), 0, Lp, Lmax, 0)
    torch.cuda.synchronize()
    return out.float()

for (L, nq, nkv, Lp, Lmax) in [(4096 + 8 * 300, 7, 1, 4096, 300), (2048, 2, 1, 2048, 0), (1000, 2, 1, 1000, 0)]:
    a = run(L, nq, nkv, Lp, Lmax, "2")
    for poly in ("0", "8"):
        b = run(L, nq, nkv, Lp, Lmax, "3", poly)
        d = (a - b).abs().view(L, nq, 128).amax(-1)  # [L, nq]
        bad = (d > 0.05).nonzero()
        print(f"L={L} nq={nq} poly={poly}: max diff {d.max().item():.4f}, bad (row,head) {bad.shape[0]}")
        if bad.shape[0]:
            rows = bad[:, 0].unique()
            print("  first bad rows", rows[:10].tolist(), "tiles", (rows // 128).unique()[:20].tolist(),
                  "heads", bad[:, 1].unique().tolist())
            print("  rows mod 128 hist", torch.bincount(rows % 128, minlength=128).nonzero().flatten()[:20].tolist())
