"""One attention launch at a given shape (for ncu source-level captures) — dev tool.
  python tools/attn_one.py L [Lp Lmax]"""
import math, pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_2507_07966_b200 import ops

L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
Lp = int(sys.argv[2]) if len(sys.argv) > 2 else None
Lmax = int(sys.argv[3]) if len(sys.argv) > 3 else 0
nq, nkv = 28, 4
qkv = torch.randn(L, (nq + 2 * nkv) * 128, device="cuda").bfloat16()
out = torch.empty(L, nq * 128, device="cuda", dtype=torch.bfloat16)
for _ in range(2):
    ops.attention(qkv, 0, qkv, nq * 128, qkv, (nq + nkv) * 128, L, nq, nq // nkv,
                  1 / math.sqrt(128), 0, Lp, Lmax, 0, out=out)
torch.cuda.synchronize()
