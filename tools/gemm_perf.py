"""Quick GEMM throughput probe (CUDA events) — dev tool, not the bench."""
import sys, pathlib, json
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_2507_07966_b200 import ops

def bench(M, N, K, epi=ops.EPI_STORE_BF16, iters=20):
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(N, K, device="cuda").bfloat16()
    out = torch.empty(M, N // 2 if epi == ops.EPI_SWIGLU_BF16 else N, device="cuda", dtype=torch.bfloat16)
    for _ in range(3): ops.gemm(A, B, epi, out=out)
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); s.record()
    for _ in range(iters): ops.gemm(A, B, epi, out=out)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / iters
    tf = 2 * M * N * K / ms / 1e9
    # cuBLAS reference point
    for _ in range(3): torch.mm(A, B.T)
    torch.cuda.synchronize(); s.record()
    for _ in range(iters): torch.mm(A, B.T)
    e.record(); torch.cuda.synchronize()
    ms2 = s.elapsed_time(e) / iters
    return dict(M=M, N=N, K=K, epi=epi, ms=round(ms, 4), tflops=round(tf, 1), cublas_tflops=round(2*M*N*K/ms2/1e9, 1))

SHAPES = [(8192, 8192, 8192, 0), (16384, 4608, 3584, 0), (16384, 3584, 3584, 0),
          (16384, 37888, 3584, 0), (16384, 3584, 18944, 0), (65536, 1152, 4608, 0),
          (16384, 37888, 3584, 4)]


if __name__ == "__main__":
    import os
    impls = sys.argv[1:] or [os.environ.get("MRSP_GEMM_IMPL", "1")]
    # impls interleaved per shape (clocks drift under the power cap)
    for M, N, K, epi in SHAPES:
        row = {"M": M, "N": N, "K": K, "epi": epi}
        for impl in impls:
            os.environ["MRSP_GEMM_IMPL"] = impl
            r = bench(M, N, K, epi)
            row[f"impl{impl}"] = r["tflops"]
            row[f"cublas_after_{impl}"] = r["cublas_tflops"]
        print(json.dumps(row), flush=True)
