"""Launch each hot kernel once at c4 shape (for `ncu --set full` captures)."""
import sys, pathlib, math
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_2507_07966_b200 import ops

which = sys.argv[1] if len(sys.argv) > 1 else "all"
L, Lp, Lmax = 131109 + 8 * 1024, 131109, 1024
if which in ("attn", "all"):
    qkv = torch.randn(L, 36 * 128, device="cuda").bfloat16()
    out = torch.empty(L, 28 * 128, device="cuda", dtype=torch.bfloat16)
    ops.attention(qkv, 0, qkv, 28 * 128, qkv, 32 * 128, L, 28, 7, 1 / math.sqrt(128), 0, Lp, Lmax, 0, out=out)
if which in ("gemm", "all"):
    A = torch.randn(16384, 3584, device="cuda").bfloat16()
    B = torch.randn(37888, 3584, device="cuda").bfloat16()
    ops.gemm(A, B, ops.EPI_SWIGLU_BF16)
torch.cuda.synchronize()
print("ok")
