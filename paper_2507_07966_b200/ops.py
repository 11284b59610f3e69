"""Thin torch-tensor front-end of the device operators in include/mrsp_c.h.

torch is used only as device-memory plumbing (allocation, streams); every
computation runs in libmrsp_b200.so. Used by the parity tests and bench.py.
"""
from __future__ import annotations

import torch

from . import _lib
from ._lib import check

EPI_STORE_BF16, EPI_BIAS_BF16, EPI_BIAS_GELU_BF16, EPI_RESID_F32, EPI_SWIGLU_BF16, EPI_STORE_F32 = range(6)


def _stream():
    return ctypes_void(torch.cuda.current_stream().cuda_stream)


def ctypes_void(x):
    return _lib.ctypes.c_void_p(int(x))


def _p(t):
    return None if t is None else ctypes_void(t.data_ptr())


def gemm(A: torch.Tensor, B: torch.Tensor, epi: int = EPI_STORE_BF16, bias=None, resid=None,
         out=None, splitk_ws=None) -> torch.Tensor:
    """C = epi(A @ B.T) on the tcgen05 GEMM. A [M,K] bf16, B [N,K] bf16.
    splitk_ws: optional device workspace (uint8) enabling split-K for M <= 128
    (mrsp_op_gemm_bf16_splitk; size from splitk_workspace_bytes(M))."""
    M, K = A.shape
    N = B.shape[0]
    assert A.dtype == torch.bfloat16 and B.dtype == torch.bfloat16 and B.shape[1] == K
    if out is None:
        if epi == EPI_RESID_F32:
            out = resid
        elif epi == EPI_STORE_F32:
            out = torch.empty(M, N, dtype=torch.float32, device=A.device)
        elif epi == EPI_SWIGLU_BF16:
            out = torch.empty(M, N // 2, dtype=torch.bfloat16, device=A.device)
        else:
            out = torch.empty(M, N, dtype=torch.bfloat16, device=A.device)
    if splitk_ws is not None:
        check(_lib.lib().mrsp_op_gemm_bf16_splitk(
            _p(A), _p(B), _p(out), M, N, K, A.stride(0), B.stride(0), out.stride(0), epi,
            _p(bias), _p(resid), resid.stride(0) if resid is not None else 0, _p(splitk_ws),
            splitk_ws.numel() * splitk_ws.element_size(), _stream()))
        return out
    check(_lib.lib().mrsp_op_gemm_bf16(
        _p(A), _p(B), _p(out), M, N, K, A.stride(0), B.stride(0), out.stride(0), epi, _p(bias),
        _p(resid), resid.stride(0) if resid is not None else 0, _stream()))
    return out


def splitk_workspace_bytes(M: int) -> int:
    return int(_lib.lib().mrsp_gemm_splitk_workspace_bytes(M))


ATTN_CAUSAL_PREFIX, ATTN_BLOCK_DIAG = 0, 1


def attention(qkv_q, q_col0, qkv_k, k_col0, qkv_v, v_col0, L, n_heads, q_per_kv, scale,
              mode=ATTN_CAUSAL_PREFIX, Lp=None, Lmax=0, blk=0, out=None, o_col0=0):
    """Flash attention over column-packed heads (see mrsp_op_attention)."""
    if out is None:
        out = torch.empty(L, n_heads * 128, dtype=torch.bfloat16, device=qkv_q.device)
    if Lp is None:
        Lp = L
    check(_lib.lib().mrsp_op_attention(
        _p(qkv_q), qkv_q.stride(0), q_col0, _p(qkv_k), qkv_k.stride(0), k_col0, _p(qkv_v),
        qkv_v.stride(0), v_col0, _p(out), out.stride(0), o_col0, L, n_heads, q_per_kv,
        float(scale), mode, Lp, Lmax, blk, _stream()))
    return out


def attention_mask(L, mode, Lp=None, Lmax=0, blk=0, device="cpu"):
    """Boolean [L, L] visibility matrix (test helper)."""
    q = torch.arange(L, device=device)[:, None]
    k = torch.arange(L, device=device)[None, :]
    if mode == ATTN_BLOCK_DIAG:
        return (q // blk) == (k // blk)
    Lp = L if Lp is None else Lp
    seg_q = torch.where(q >= Lp, (q - Lp) // max(Lmax, 1), -1)
    seg_k = torch.where(k >= Lp, (k - Lp) // max(Lmax, 1), -2)
    return (k <= q) & ((k < Lp) | (seg_q == seg_k))
