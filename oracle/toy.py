"""ctypes front-end of oracle/mrsp_oracle.c — the CPU restatement of the
reference's toy MR-SP path. TEST INFRASTRUCTURE: imported only by tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline legs, never by the
product package.
"""
from __future__ import annotations

import ctypes
import pathlib
import subprocess

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
SO = HERE / "_build" / "liboracle.so"

_l = None
_d = ctypes.POINTER(ctypes.c_double)
_u64 = ctypes.POINTER(ctypes.c_uint64)
_i32 = ctypes.POINTER(ctypes.c_int32)


def lib():
    global _l
    if _l is None:
        if not SO.exists():
            subprocess.run(["make", "-C", str(HERE), "all"], check=True, capture_output=True)
        l = ctypes.CDLL(str(SO))
        l.oracle_substream_seed.restype = ctypes.c_uint64
        l.oracle_substream_seed.argtypes = [ctypes.c_uint64, ctypes.c_char_p]
        l.oracle_substream_draws.argtypes = [ctypes.c_uint64, ctypes.c_char_p, _u64, ctypes.c_int]
        l.oracle_rng_uniform.argtypes = [ctypes.c_uint64, _d, ctypes.c_long]
        l.oracle_plan_shards.argtypes = [ctypes.c_uint64, ctypes.c_int, _u64]
        l.oracle_gen_video.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_int, _d]
        l.oracle_encoder_generate.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_int, _d]
        l.oracle_policy_param_count.restype = ctypes.c_long
        l.oracle_policy_param_count.argtypes = [ctypes.c_int] * 3
        l.oracle_policy_random.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_uint64,
                                           ctypes.c_double, _d]
        l.oracle_serial_encode.argtypes = [_d, ctypes.c_int, ctypes.c_int, _d, ctypes.c_long, _d]
        l.oracle_step_logits.argtypes = [_d, ctypes.c_int, ctypes.c_int, ctypes.c_int, _d,
                                         ctypes.c_int, _d]
        l.oracle_serial_prefill.argtypes = [_d, ctypes.c_int, ctypes.c_int, ctypes.c_int, _d, _i32,
                                            _u64, ctypes.c_long, ctypes.c_long, _d]
        l.oracle_log_softmax.argtypes = [_d, ctypes.c_int, _d]
        l.oracle_context_vector.argtypes = [_d, ctypes.c_int, ctypes.c_int, _d, ctypes.c_long, _i32,
                                            ctypes.c_long, _d]
        _l64 = ctypes.POINTER(ctypes.c_long)
        l.oracle_grpo_gradient.argtypes = [_d, _d, ctypes.c_int, ctypes.c_int, ctypes.c_int, _d,
                                           ctypes.c_long, _i32, ctypes.c_long, _i32, _l64,
                                           ctypes.c_long, _d, _d, ctypes.c_double,
                                           ctypes.c_double, ctypes.c_int, _d, _d]
        l.oracle_sft_loss_and_grad.argtypes = [_d, ctypes.c_int, ctypes.c_int, ctypes.c_int, _d,
                                               ctypes.c_long, _i32, ctypes.c_long, _i32,
                                               ctypes.c_long, _d, _d]
        _l = l
    return _l


def _p(a, t=ctypes.c_double):
    return a.ctypes.data_as(ctypes.POINTER(t))


def substream_draws(base: int, tag: str, n: int) -> np.ndarray:
    out = np.zeros(n, dtype=np.uint64)
    lib().oracle_substream_draws(base, tag.encode(), _p(out, ctypes.c_uint64), n)
    return out


def uniform(seed: int, n: int) -> np.ndarray:
    out = np.zeros(n)
    lib().oracle_rng_uniform(seed, _p(out), n)
    return out


def plan_shards(n: int, k: int):
    out = np.zeros(2 * max(k, 1), dtype=np.uint64)
    if lib().oracle_plan_shards(n, k, _p(out, ctypes.c_uint64)):
        raise ValueError("plan_shards: sp_degree must be >= 1")
    return [(int(out[2 * i]), int(out[2 * i + 1])) for i in range(k)]


def gen_video(seed: int, frames: int, feature_dim: int) -> np.ndarray:
    out = np.zeros((frames, feature_dim))
    if lib().oracle_gen_video(seed, frames, feature_dim, _p(out)):
        raise ValueError("gen_video: bad arguments")
    return out


def video_id(seed: int, frames: int) -> str:
    return f"v{seed}f{frames}"  # mmseq.cpp:64


def encoder_generate(seed: int, d: int, p: int) -> np.ndarray:
    w = np.zeros((d, p))
    if lib().oracle_encoder_generate(seed, d, p, _p(w)):
        raise ValueError("EncoderParams: d >= 1 and p >= 4 required")
    return w


def policy_random(V: int, d: int, h: int, seed: int, scale: float) -> np.ndarray:
    theta = np.zeros(lib().oracle_policy_param_count(V, d, h))
    lib().oracle_policy_random(V, d, h, seed, scale, _p(theta))
    return theta


def serial_encode(w: np.ndarray, frames: np.ndarray) -> np.ndarray:
    d, p = w.shape
    frames = np.ascontiguousarray(frames, dtype=np.float64)
    out = np.zeros((frames.shape[0], d))
    lib().oracle_serial_encode(_p(np.ascontiguousarray(w)), d, p, _p(frames), frames.shape[0], _p(out))
    return out


def step_logits(theta, V, d, h, ctx, prev) -> np.ndarray:
    out = np.zeros(V)
    ctx = np.ascontiguousarray(ctx, dtype=np.float64)
    if lib().oracle_step_logits(_p(theta), V, d, h, _p(ctx), prev, _p(out)):
        raise ValueError("step_logits: prev token out of range")
    return out


def serial_prefill(theta, V, d, h, contexts, rows, lengths):
    contexts = np.ascontiguousarray(contexts, dtype=np.float64)
    rows = np.ascontiguousarray(rows, dtype=np.int32)
    lengths = np.ascontiguousarray(lengths, dtype=np.uint64)
    out = np.zeros((int(lengths.sum()), V))
    rc = lib().oracle_serial_prefill(_p(theta), V, d, h, _p(contexts), _p(rows, ctypes.c_int32),
                                     _p(lengths, ctypes.c_uint64), rows.shape[0], rows.shape[1],
                                     _p(out))
    if rc:
        raise ValueError("step_logits: prev token out of range")
    return out


def log_softmax(x) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.zeros_like(x)
    lib().oracle_log_softmax(_p(x), x.shape[0], _p(out))
    return out


def context_vector(theta, V, d, frame_emb, text):
    frame_emb = np.ascontiguousarray(frame_emb, dtype=np.float64)
    text = np.ascontiguousarray(text, dtype=np.int32)
    out = np.zeros(d)
    if lib().oracle_context_vector(_p(theta), V, d, _p(frame_emb), frame_emb.shape[0],
                                   _p(text, ctypes.c_int32), text.shape[0], _p(out)):
        raise ValueError("context_vector: bad input")
    return out


def grpo_gradient(theta, ref, V, d, h, frame_emb, text, tokens, old_logprobs, advantages,
                  clip_eps=0.2, kl_beta=0.04, sampled_kl=False):
    """grpo_gradient (grpo.cpp:122-206) -> (grad, stats dict). `tokens` and
    `old_logprobs` are per-rollout lists."""
    frame_emb = np.ascontiguousarray(frame_emb, dtype=np.float64).reshape(-1, d)
    text = np.ascontiguousarray(text, dtype=np.int32)
    lens = np.array([len(t) for t in tokens], dtype=np.int64)
    tok = np.ascontiguousarray(np.concatenate([np.asarray(t, dtype=np.int32) for t in tokens]))
    old = np.ascontiguousarray(np.concatenate([np.asarray(o, dtype=np.float64)
                                               for o in old_logprobs]))
    adv = np.ascontiguousarray(advantages, dtype=np.float64)
    theta = np.ascontiguousarray(theta, dtype=np.float64)
    ref = np.ascontiguousarray(ref, dtype=np.float64)
    grad = np.zeros(theta.shape[0])
    st = np.zeros(4)
    if lib().oracle_grpo_gradient(_p(theta), _p(ref), V, d, h, _p(frame_emb), frame_emb.shape[0],
                                  _p(text, ctypes.c_int32), text.shape[0],
                                  _p(tok, ctypes.c_int32), _p(lens, ctypes.c_long), lens.shape[0],
                                  _p(old), _p(adv), clip_eps, kl_beta, int(sampled_kl), _p(grad),
                                  _p(st)):
        raise ValueError("grpo_gradient: bad input")
    return grad, {"objective": st[0], "mean_kl": st[1], "clip_fraction": st[2],
                  "token_count": int(st[3])}


def sft_loss_and_grad(theta, V, d, h, frame_emb, text, targets):
    """sft_loss_and_grad (grpo.cpp:208-223) -> (loss, grad)."""
    frame_emb = np.ascontiguousarray(frame_emb, dtype=np.float64).reshape(-1, d)
    text = np.ascontiguousarray(text, dtype=np.int32)
    tg = np.ascontiguousarray(targets, dtype=np.int32)
    theta = np.ascontiguousarray(theta, dtype=np.float64)
    grad = np.zeros(theta.shape[0])
    loss = np.zeros(1)
    if lib().oracle_sft_loss_and_grad(_p(theta), V, d, h, _p(frame_emb), frame_emb.shape[0],
                                      _p(text, ctypes.c_int32), text.shape[0],
                                      _p(tg, ctypes.c_int32), tg.shape[0], _p(loss), _p(grad)):
        raise ValueError("sft_loss_and_grad: bad input")
    return float(loss[0]), grad
