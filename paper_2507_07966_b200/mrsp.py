"""Python mirror of the reference's lvrl::mrsp interface (engine.hpp:17-157),
over the C-ABI. Same names, argument meaning and error behaviour, so the
parity tests read like the reference's own tests (proj/tests/test_engine.cpp).

Arrays are numpy (host). The toy model path is fp64 and bit-identical to the
reference CPU (csrc/toy.cu).
"""
from __future__ import annotations

import threading
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from ._lib import GatherError, InvalidArgument, c_f64p, c_i32p, c_u64p, check, ptr

K_PAD = 0  # mmseq.hpp:15
K_EOS = 1  # mmseq.hpp:16


@dataclass
class ShardPlan:
    """engine.hpp:20-23: contiguous [begin, end) ranges + total."""
    ranges: List[Tuple[int, int]]
    total: int


def plan_shards(n_items: int, sp_degree: int) -> ShardPlan:
    """engine.cpp:15-29 via mrsp_plan_shards."""
    k = int(sp_degree)
    buf = np.zeros(max(2 * k, 2), dtype=np.uint64)
    check(_lib.lib().mrsp_plan_shards(int(n_items), k, ptr(buf, _lib.ctypes.c_uint64)))
    return ShardPlan([(int(buf[2 * w]), int(buf[2 * w + 1])) for w in range(k)], int(n_items))


def _flat(plan: ShardPlan) -> np.ndarray:
    return np.array([x for r in plan.ranges for x in r], dtype=np.uint64)


class EngineStats:
    """engine.hpp:27-41 (relaxed atomics upstream; a lock here)."""

    FIELDS = ("encoder_invocations", "cache_hits", "cache_misses", "gather_bytes", "pad_reads")

    def __init__(self):
        self._mu = threading.Lock()
        self.reset()

    def reset(self):
        for f in self.FIELDS:
            setattr(self, f, 0)

    def add(self, name: str, n: int):
        with self._mu:
            setattr(self, name, getattr(self, name) + int(n))


@dataclass
class EncodedSlice:
    """engine.hpp:43-48."""
    worker: int
    begin: int
    end: int
    embeddings: np.ndarray  # (end-begin, d) float64


@dataclass
class PaddedBatch:
    """engine.hpp:50-61."""
    rows: np.ndarray        # (n_rows, max_len) int32, PAD-filled
    lengths: np.ndarray     # (n_rows,) uint64
    max_len: int

    def at(self, row: int, pos: int, stats: Optional[EngineStats]) -> int:
        if pos >= int(self.lengths[row]) and stats is not None:
            stats.add("pad_reads", 1)
        return int(self.rows[row, pos])


def pad_batch(sequences: Sequence[Sequence[int]], pad: int = K_PAD) -> PaddedBatch:
    """engine.cpp:31-43."""
    if len(sequences) == 0:
        raise InvalidArgument(1, "pad_batch: empty batch")
    max_len = max((len(s) for s in sequences), default=0)
    rows = np.full((len(sequences), max_len), pad, dtype=np.int32)
    for i, s in enumerate(sequences):
        rows[i, : len(s)] = np.asarray(s, dtype=np.int32)
    return PaddedBatch(rows, np.array([len(s) for s in sequences], dtype=np.uint64), max_len)


def unpad_batch(batch: PaddedBatch) -> List[List[int]]:
    """engine.cpp:45-50."""
    return [batch.rows[i, : int(batch.lengths[i])].tolist() for i in range(batch.rows.shape[0])]


@dataclass
class EncoderParams:
    """policy.hpp:17-23: W is d x p row-major."""
    d: int
    p: int
    w: np.ndarray


@dataclass
class PolicyParams:
    """policy.hpp:27-56: flat theta E_txt|A|B|c|U|b."""
    V: int
    d: int
    h: int
    theta: np.ndarray


def _encode(enc: EncoderParams, frames: np.ndarray, ranges: np.ndarray, k: int):
    frames = np.ascontiguousarray(frames, dtype=np.float64)
    n = frames.shape[0]
    if frames.ndim != 2 or (n and frames.shape[1] != enc.p):
        raise InvalidArgument(1, "encode_frame: frame dimension mismatch")
    out = np.empty((n, enc.d), dtype=np.float64)
    items = np.zeros(k, dtype=np.uint64)
    w = np.ascontiguousarray(enc.w, dtype=np.float64)
    check(_lib.lib().mrsp_toy_encode(k, ptr(w, _lib.ctypes.c_double), enc.d, enc.p,
                                     ptr(frames, _lib.ctypes.c_double), n,
                                     ptr(ranges, _lib.ctypes.c_uint64),
                                     ptr(out, _lib.ctypes.c_double),
                                     ptr(items, _lib.ctypes.c_uint64)))
    return out, items


def serial_encode(enc: EncoderParams, frames: np.ndarray) -> np.ndarray:
    """engine.cpp:52-57 (one rank, one range)."""
    out, _ = _encode(enc, frames, np.array([0, frames.shape[0]], dtype=np.uint64), 1)
    return out


def _prefill(params: PolicyParams, contexts: np.ndarray, batch: PaddedBatch, ranges: np.ndarray,
             k: int):
    ctx = np.ascontiguousarray(contexts, dtype=np.float64)
    rows = np.ascontiguousarray(batch.rows, dtype=np.int32)
    lengths = np.ascontiguousarray(batch.lengths, dtype=np.uint64)
    total = int(lengths.sum())
    out = np.empty((total, params.V), dtype=np.float64)
    pad_reads = np.zeros(1, dtype=np.uint64)
    theta = np.ascontiguousarray(params.theta, dtype=np.float64)
    check(_lib.lib().mrsp_toy_prefill(
        k, ptr(theta, _lib.ctypes.c_double), params.V, params.d, params.h,
        ptr(ctx, _lib.ctypes.c_double), ptr(rows, _lib.ctypes.c_int32),
        ptr(lengths, _lib.ctypes.c_uint64), rows.shape[0], batch.max_len,
        ptr(ranges, _lib.ctypes.c_uint64), ptr(out, _lib.ctypes.c_double),
        ptr(pad_reads, _lib.ctypes.c_uint64)))
    split = np.cumsum(lengths.astype(np.int64))[:-1]
    return np.split(out, split), int(pad_reads[0])


def serial_prefill(params: PolicyParams, contexts: np.ndarray, batch: PaddedBatch):
    """engine.cpp:59-71: list over rows of (len_r, V) logits."""
    if len(contexts) != batch.rows.shape[0]:
        raise InvalidArgument(1, "serial_prefill: one context per row required")
    out, _ = _prefill(params, contexts, batch, np.array([0, batch.max_len], dtype=np.uint64), 1)
    return out


class WorkerGroup:
    """engine.hpp:75-99. Ranks are CUDA streams on the current device."""

    def __init__(self, sp_degree: int, enc: EncoderParams):
        if sp_degree < 1:
            raise InvalidArgument(1, "WorkerGroup: sp_degree must be >= 1")
        self._k = int(sp_degree)
        self._enc = enc
        self._stats = EngineStats()

    def degree(self) -> int:
        return self._k

    def encoder(self, worker: int) -> EncoderParams:
        if not 0 <= worker < self._k:
            raise IndexError("WorkerGroup::encoder")
        return self._enc

    def stats(self) -> EngineStats:
        return self._stats

    def parallel_encode(self, frames: np.ndarray, plan: ShardPlan) -> List[EncodedSlice]:
        """engine.cpp:78-101."""
        if plan.total != frames.shape[0]:
            raise InvalidArgument(1, "parallel_encode: plan does not cover the video frames")
        if len(plan.ranges) != self._k:
            raise InvalidArgument(1, "parallel_encode: plan degree mismatch")
        out, items = _encode(self._enc, frames, _flat(plan), self._k)
        self._stats.add("encoder_invocations", int(items.sum()))
        return [EncodedSlice(w, b, e, out[b:e]) for w, (b, e) in enumerate(plan.ranges)]

    def parallel_prefill(self, params: PolicyParams, contexts: np.ndarray, batch: PaddedBatch,
                         plan: ShardPlan):
        """engine.cpp:103-130."""
        if plan.total != batch.max_len:
            raise InvalidArgument(1, "parallel_prefill: plan does not cover the padded length")
        if len(plan.ranges) != self._k:
            raise InvalidArgument(1, "parallel_prefill: plan degree mismatch")
        if len(contexts) != batch.rows.shape[0]:
            raise InvalidArgument(1, "parallel_prefill: one context per row required")
        out, pad_reads = _prefill(params, contexts, batch, _flat(plan), self._k)
        self._stats.add("pad_reads", pad_reads)
        return out


def all_gather(slices: List[EncodedSlice], sp_degree: int,
               stats: Optional[EngineStats]) -> np.ndarray:
    """engine.cpp:132-153: order-independent concatenation + simulated bytes."""
    if not slices:
        raise GatherError(2, "all_gather: no slices")
    ordered = sorted(slices, key=lambda s: s.begin)
    expect, parts, values = 0, [], 0
    for s in ordered:
        if s.begin != expect:
            raise GatherError(2, "all_gather: missing or overlapping slice")
        if s.embeddings.shape[0] != s.end - s.begin:
            raise GatherError(2, "all_gather: slice length mismatch")
        expect = s.end
        parts.append(s.embeddings)
        values += s.embeddings.size
    if stats is not None:
        stats.add("gather_bytes", values * (sp_degree - 1) * 8)
    return np.concatenate(parts, axis=0) if parts else np.zeros((0, 0))


class EmbeddingCache:
    """engine.hpp:110-128 / engine.cpp:155-197: exactly-once fill per video id."""

    class _Entry:
        def __init__(self):
            self.cv = threading.Condition()
            self.ready = False
            self.value = None
            self.error = None  # set when the fill raised

    def __init__(self):
        self._mu = threading.Lock()
        self._map: Dict[str, "EmbeddingCache._Entry"] = {}

    def get_or_encode(self, group: WorkerGroup, video_id: str, frames: np.ndarray,
                      plan: ShardPlan):
        with self._mu:
            entry = self._map.get(video_id)
            filler = entry is None
            if filler:
                entry = self._map[video_id] = EmbeddingCache._Entry()
                group.stats().add("cache_misses", 1)
            else:
                group.stats().add("cache_hits", 1)
        if filler:
            try:
                value = all_gather(group.parallel_encode(frames, plan), group.degree(),
                                   group.stats())
            except BaseException as exc:
                # publish the failure: drop the key (a later call retries) and
                # wake the waiters, which re-raise instead of blocking forever
                with self._mu:
                    if self._map.get(video_id) is entry:
                        del self._map[video_id]
                with entry.cv:
                    entry.error, entry.ready = exc, True
                    entry.cv.notify_all()
                raise
            value.setflags(write=False)
            with entry.cv:
                entry.value, entry.ready = value, True
                entry.cv.notify_all()
            return value, False
        with entry.cv:
            entry.cv.wait_for(lambda: entry.ready)
            if entry.error is not None:
                raise RuntimeError(f"EmbeddingCache: encoding {video_id} failed in another "
                                   f"caller") from entry.error
            return entry.value, True

    def size(self) -> int:
        with self._mu:
            return len(self._map)

    def clear(self) -> None:
        with self._mu:
            self._map.clear()


# ---- backward: grpo.hpp:14-62 ----

@dataclass
class MultimodalSequence:
    """mmseq.hpp: the frame embeddings (n_frames x d) + the question's text tokens."""
    frame_embeddings: np.ndarray
    text_tokens: Sequence[int]


@dataclass
class Rollout:
    """policy.hpp: sampled tokens + the log-probs recorded while sampling."""
    tokens: Sequence[int]
    old_logprobs: Sequence[float]


@dataclass
class RolloutGroup:
    """grpo.hpp:34-38 (advantages = Advantages::values)."""
    rollouts: List[Rollout]
    advantages: Sequence[float]
    sample_id: str = ""


@dataclass
class GrpoConfig:
    """grpo.hpp:14-23 (the fields the objective and gradient read)."""
    clip_eps: float = 0.2
    kl_beta: float = 0.04
    sampled_kl: bool = False


@dataclass
class GroupStats:
    """grpo.hpp:40-45."""
    objective: float = 0.0
    mean_kl: float = 0.0
    clip_fraction: float = 0.0
    token_count: int = 0


def _seq_arrays(params: PolicyParams, seq: MultimodalSequence):
    fe = np.ascontiguousarray(seq.frame_embeddings, dtype=np.float64).reshape(-1, params.d)
    text = np.ascontiguousarray(np.asarray(seq.text_tokens, dtype=np.int32))
    return fe, text


def grpo_gradient(group: RolloutGroup, theta: PolicyParams, ref: PolicyParams,
                  seq: MultimodalSequence, cfg: GrpoConfig, sp_degree: int = 1):
    """grpo.cpp:122-206 on the device -> (grad, GroupStats). The positions run
    sharded over `sp_degree` ranks (plan_shards over the longest rollout)."""
    if not group.rollouts:
        raise InvalidArgument(1, "grpo: empty rollout group")
    for r in group.rollouts:
        if len(r.tokens) == 0:
            raise InvalidArgument(1, "grpo: empty rollout")
        if len(r.old_logprobs) != len(r.tokens):
            raise InvalidArgument(1, "grpo: old_logprobs missing")
    if (theta.V, theta.d, theta.h) != (ref.V, ref.d, ref.h):
        raise InvalidArgument(1, "kl_per_position: vocab mismatch")
    fe, text = _seq_arrays(theta, seq)
    lens = np.array([len(r.tokens) for r in group.rollouts], dtype=np.uint64)
    tok = np.ascontiguousarray(np.concatenate([np.asarray(r.tokens, dtype=np.int32)
                                               for r in group.rollouts]))
    old = np.ascontiguousarray(np.concatenate([np.asarray(r.old_logprobs, dtype=np.float64)
                                               for r in group.rollouts]))
    adv = np.ascontiguousarray(np.asarray(group.advantages, dtype=np.float64))
    if adv.shape[0] != len(group.rollouts):
        raise InvalidArgument(1, "grpo: one advantage per rollout required")
    th = np.ascontiguousarray(theta.theta, dtype=np.float64)
    rf = np.ascontiguousarray(ref.theta, dtype=np.float64)
    ranges = _flat(plan_shards(int(lens.max()), sp_degree))
    grad = np.empty(th.shape[0])
    st = np.zeros(4)
    c = _lib.ctypes
    check(_lib.lib().mrsp_toy_grpo_gradient(
        sp_degree, ptr(th, c.c_double), ptr(rf, c.c_double), theta.V, theta.d, theta.h,
        ptr(fe, c.c_double), fe.shape[0], ptr(text, c.c_int32), text.shape[0],
        ptr(tok, c.c_int32), ptr(lens, c.c_uint64), lens.shape[0], ptr(old, c.c_double),
        ptr(adv, c.c_double), cfg.clip_eps, cfg.kl_beta, int(cfg.sampled_kl),
        ptr(ranges, c.c_uint64), ptr(grad, c.c_double), ptr(st, c.c_double)))
    return grad, GroupStats(float(st[0]), float(st[1]), float(st[2]), int(st[3]))


def sft_loss_and_grad(theta: PolicyParams, seq: MultimodalSequence,
                      target_tokens: Sequence[int], sp_degree: int = 1):
    """grpo.cpp:208-223 on the device -> (loss, grad)."""
    if len(target_tokens) == 0:
        raise InvalidArgument(1, "sft_loss_and_grad: empty targets")
    fe, text = _seq_arrays(theta, seq)
    tg = np.ascontiguousarray(np.asarray(target_tokens, dtype=np.int32))
    th = np.ascontiguousarray(theta.theta, dtype=np.float64)
    ranges = _flat(plan_shards(tg.shape[0], sp_degree))
    grad = np.empty(th.shape[0])
    loss = np.zeros(1)
    c = _lib.ctypes
    check(_lib.lib().mrsp_toy_sft_loss_and_grad(
        sp_degree, ptr(th, c.c_double), theta.V, theta.d, theta.h, ptr(fe, c.c_double),
        fe.shape[0], ptr(text, c.c_int32), text.shape[0], ptr(tg, c.c_int32), tg.shape[0],
        ptr(ranges, c.c_uint64), ptr(loss, c.c_double), ptr(grad, c.c_double)))
    return float(loss[0]), grad
