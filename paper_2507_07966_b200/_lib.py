"""ctypes binding of libmrsp_b200.so (include/mrsp_c.h).

The library is built in-tree by ``paper_2507_07966_b200/csrc/Makefile`` (see
``__graft_entry__.build``). There is no fallback: if the shared object is
missing, importing the engine raises.
"""
from __future__ import annotations

import ctypes
import os
import pathlib

_HERE = pathlib.Path(__file__).resolve().parent
LIB_PATH = _HERE / "_lib" / "libmrsp_b200.so"

c_u64p = ctypes.POINTER(ctypes.c_uint64)
c_i32p = ctypes.POINTER(ctypes.c_int32)
c_f64p = ctypes.POINTER(ctypes.c_double)
c_f32p = ctypes.POINTER(ctypes.c_float)

STATUS = {
    0: "MRSP_OK",
    1: "MRSP_INVALID_ARGUMENT",
    2: "MRSP_RUNTIME_ERROR",
    3: "MRSP_OUT_OF_RANGE",
    4: "MRSP_LOGIC_ERROR",
    5: "MRSP_CUDA_ERROR",
    6: "MRSP_NCCL_ERROR",
    7: "MRSP_OUT_OF_MEMORY",
    8: "MRSP_NO_DEVICE",
}


class MrspError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.msg = msg


class InvalidArgument(MrspError, ValueError):
    """Mirrors std::invalid_argument (engine.cpp:16, :32, :74, :80-83, :107-112)."""


class GatherError(MrspError):
    """Mirrors std::runtime_error from all_gather (engine.cpp:133-142)."""


_lib = None

# (name, restype, argtypes) for every symbol include/mrsp_c.h declares.
SIGNATURES: dict = {}


def _sig(name, argtypes, restype=ctypes.c_int):
    SIGNATURES[name] = (restype, argtypes)


_sig("mrsp_last_error", [], ctypes.c_char_p)
_sig("mrsp_version", [], ctypes.c_char_p)
_sig("mrsp_device_count", [], ctypes.c_int)
_sig("mrsp_launch_count", [], ctypes.c_uint64)
_sig("mrsp_plan_shards", [ctypes.c_uint64, ctypes.c_int, c_u64p])
_sig("mrsp_toy_encode", [ctypes.c_int, c_f64p, ctypes.c_int, ctypes.c_int, c_f64p, ctypes.c_uint64,
                         c_u64p, c_f64p, c_u64p])
_sig("mrsp_toy_prefill", [ctypes.c_int, c_f64p, ctypes.c_int, ctypes.c_int, ctypes.c_int, c_f64p,
                          c_i32p, c_u64p, ctypes.c_uint64, ctypes.c_uint64, c_u64p, c_f64p, c_u64p])
_sig("mrsp_toy_grpo_gradient", [ctypes.c_int, c_f64p, c_f64p, ctypes.c_int, ctypes.c_int,
                                ctypes.c_int, c_f64p, ctypes.c_uint64, c_i32p, ctypes.c_uint64,
                                c_i32p, c_u64p, ctypes.c_uint64, c_f64p, c_f64p, ctypes.c_double,
                                ctypes.c_double, ctypes.c_int, c_u64p, c_f64p, c_f64p])
_sig("mrsp_toy_sft_loss_and_grad", [ctypes.c_int, c_f64p, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_int, c_f64p, ctypes.c_uint64, c_i32p,
                                    ctypes.c_uint64, c_i32p, ctypes.c_uint64, c_u64p, c_f64p,
                                    c_f64p])
_sig("mrsp_op_gemm_bf16", [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                           ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                           ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                           ctypes.c_void_p])
_sig("mrsp_op_gemm_bf16_splitk", [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                  ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p])
_sig("mrsp_gemm_splitk_workspace_bytes", [ctypes.c_int], ctypes.c_size_t)
_sig("mrsp_op_attention", [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                           ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                           ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                           ctypes.c_float, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                           ctypes.c_void_p])
_V, _I, _F, _U64, _I64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_float, ctypes.c_uint64, ctypes.c_int64
_sig("mrsp_gen_video", [_U64, _I, _I, c_f32p])
_sig("mrsp_lmhead_workspace_bytes", [_I, _I], ctypes.c_size_t)
_sig("mrsp_op_lmhead_logprob", [_V, _I, _V, _I, _I, _I, _V, _V, _V, _V, ctypes.c_size_t, _V])
_sig("mrsp_op_rmsnorm", [_V, _I, _V, _V, _I, _I, _I, _F, _V, _V])
_sig("mrsp_op_layernorm", [_V, _I, _V, _V, _V, _I, _I, _I, _F, _V])
_sig("mrsp_op_rope", [_V, _I, _I, _I, _V, _I, _F, _V])
_sig("mrsp_op_patchify", [_V, _V, _I, _I, _I, _I, _I, _V])
_sig("mrsp_op_pack_sequence", [_V, _I, _V, _I, _V, _V, _I, _V, _I, _I64, _I, _V, _V, _V, _V, _V])
_sig("mrsp_nccl_unique_id", [_V])
_sig("mrsp_ulysses_plan", [_I, _I, _I, _I, _V])
_sig("mrsp_attn_row_part", [_I, _I, _I], ctypes.c_int)
_sig("mrsp_head_split", [_I, _I, _I, _I, _I, _V])
_sig("mrsp_engine_create", [_V, _I, _I, _I, _U64, _U64, _U64, _I, _V, _V])
_sig("mrsp_engine_destroy", [_V])
_sig("mrsp_engine_encode", [_V, ctypes.c_char_p, _V, _I, _I, _I, _V])
_sig("mrsp_engine_prefill_logprobs", [_V, ctypes.c_char_p, _V, _I, _V, _V, _I, _I, _I, _V, _V, _I])
_sig("mrsp_engine_step", [_V, ctypes.c_char_p, _V, _I, _I, _I, _V, _I, _V, _V, _I, _I, _V, _V, _V, _I])
_sig("mrsp_lmhead_dual_workspace_bytes", [_I, _I], ctypes.c_size_t)
_sig("mrsp_op_grpo_stats", [_V, _V, _V, _V, _V, _V, _I, ctypes.c_double, ctypes.c_double, _I, _V, _V])
_sig("mrsp_op_lmhead_dual", [_V, _V, _V, _V, _I, _I, _I, _V, _V, _V, _V, _V, ctypes.c_size_t, _V])
_sig("mrsp_engine_stats", [_V, _V, _I])
_sig("mrsp_engine_cache", [_V, _I, _I, _V])
_sig("mrsp_engine_get_embeddings", [_V, ctypes.c_char_p, _V, ctypes.c_size_t, _V])
_sig("mrsp_engine_profile", [_V, _I, _I, _V, _V])
_sig("mrsp_engine_stream", [_V], ctypes.c_void_p)
_sig("mrsp_p2p_blob_bytes", [], ctypes.c_size_t)
_sig("mrsp_engine_save_weights", [_V, ctypes.c_char_p])
_sig("mrsp_engine_generate", [_V, ctypes.c_char_p, _V, _I, _I, _I, _F, _U64, _V, _V, _V])
_sig("mrsp_engine_load_weights", [_V, ctypes.c_char_p, _I, ctypes.c_char_p])
_sig("mrsp_engine_cache_save", [_V, ctypes.c_char_p, ctypes.c_char_p])
_sig("mrsp_engine_cache_load", [_V, ctypes.c_char_p, ctypes.c_char_p, _V])
_sig("mrsp_engine_p2p_export", [_V, _I, ctypes.c_long, ctypes.c_long, _V])
_sig("mrsp_engine_p2p_import", [_V, _V])
# backward pass
_sig("mrsp_op_gemm_bf16_mn", [_V, _V, _V, _I, _I, _I, _I, _I, _I, _I, _I, _I, _V, _V, _I, _V])
_sig("mrsp_op_attention_lse", [_V, _I, _I, _V, _I, _I, _V, _I, _I, _V, _I, _I, _I, _I, _I, _F,
                               _I, _I, _V, _I, _V])
_sig("mrsp_op_attention_bwd", [_V, _I, _I, _I, _I, _V, _I, _V, _I, _V, _V, _I, _V, _I, _I, _I, _I,
                               _F, _I, _I, _V])
_sig("mrsp_op_rmsnorm_bwd", [_V, _I, _V, _V, _I, _V, _I, _I, _I, _F, _V, _V, _V])
_sig("mrsp_op_gemm_swiglu_bwd", [_V, _V, _V, _V, _V, _I, _I, _I, _V])
_sig("mrsp_op_lmhead_dual_dlogits", [_V, _V, _V, _V, _I, _I, _I, _V, _V, _F, _V, _V, _V, _V, _I,
                                     _V])
_sig("mrsp_engine_grpo_backward", [_V, ctypes.c_char_p, _V, _I, _V, _V, _I, _I, _V, _V,
                                   ctypes.c_double, ctypes.c_double, _I, _V, _V])
_sig("mrsp_engine_save_grads", [_V, ctypes.c_char_p])
_sig("mrsp_engine_sft_backward", [_V, ctypes.c_char_p, _V, _I, _V, _V, _I, _I, _V, _V])


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                " (the B200 engine has no CPU fallback)")
        # libcudart / libcuda come from the CUDA toolkit or torch's bundle.
        l = ctypes.CDLL(str(LIB_PATH), mode=ctypes.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(l, name)
            fn.restype = res
            fn.argtypes = args
        _lib = l
    return _lib


def check(status: int) -> None:
    if status == 0:
        return
    msg = lib().mrsp_last_error().decode()
    if status == 1:
        raise InvalidArgument(status, msg)
    if status == 2 and msg.startswith("all_gather"):
        raise GatherError(status, msg)
    raise MrspError(status, msg)


def ptr(arr, ctype):
    """Pointer to a C-contiguous numpy array's data."""
    assert arr.flags["C_CONTIGUOUS"], "array must be C-contiguous"
    return arr.ctypes.data_as(ctypes.POINTER(ctype))


def device_count() -> int:
    return int(lib().mrsp_device_count())


os.environ.setdefault("CUDA_MODULE_LOADING", "LAZY")
