"""Host-side front-end of the MR-SP engine (include/mrsp_c.h, csrc/engine.cu).

Mirrors the reference's two-stage call sites: ``encode`` is the Stage-1
fetch_embeddings / EmbeddingCache::get_or_encode (grpo.cpp:289-295,
engine.cpp:155-197); ``prefill_logprobs`` is engine_group_logits + the
log-softmax/gather (grpo.cpp:44-55, :82-85); ``step`` is run_step
(engine.cpp:203-225). All compute runs in libmrsp_b200.so.
"""
from __future__ import annotations

import ctypes
from dataclasses import asdict, dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import check

K_PAD, K_EOS, K_CONTENT_BASE = 0, 1, 10  # mmseq.hpp:15-23


class ModelConfig(ctypes.Structure):
    """mrsp_model_config."""
    _fields_ = [(n, ctypes.c_int) for n in (
        "image_size", "patch", "v_dim", "v_heads", "v_head_dim", "v_mlp", "v_layers", "dim",
        "n_q_heads", "n_kv_heads", "head_dim", "mlp", "layers", "vocab")] + [
        ("rope_theta", ctypes.c_float), ("rms_eps", ctypes.c_float), ("ln_eps", ctypes.c_float)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}

    @property
    def tokens_per_frame(self) -> int:
        return (self.image_size // self.patch) ** 2


def _cfg(**kw) -> ModelConfig:
    base = dict(rope_theta=1e6, rms_eps=1e-6, ln_eps=1e-6, head_dim=128)
    base.update(kw)
    return ModelConfig(**base)


SIGLIP = dict(image_size=224, patch=14, v_dim=1152, v_heads=16, v_head_dim=72, v_mlp=4304,
              v_layers=27)
QWEN7B = dict(dim=3584, n_q_heads=28, n_kv_heads=4, mlp=18944, layers=28, vocab=152064)


@dataclass
class Workload:
    """One BASELINE.json configuration: model shape + the synthetic GRPO group."""
    name: str
    cfg: ModelConfig
    frames: int
    sp: int
    G: int
    n_question: int
    len_lo: int
    len_hi: int
    desc: str = ""


def workloads():
    """BASELINE.json configs c1..c5."""
    c1 = _cfg(image_size=64, patch=8, v_dim=256, v_heads=4, v_head_dim=64, v_mlp=1024, v_layers=2,
              dim=256, n_q_heads=4, n_kv_heads=2, mlp=1024, layers=2, vocab=32)
    c2 = _cfg(**SIGLIP, **{**QWEN7B, "layers": 4})
    c3 = _cfg(**SIGLIP, **QWEN7B)
    return {
        "c1": Workload("c1", c1, 8, 1, 4, 3, 6, 12,
                       "tiny synthetic MR-SP step: 8 frames x 64 tokens, 2-layer vision + 2-layer "
                       "LLM (d=256), SP=1, 4 rollouts"),
        "c2": Workload("c2", c2, 64, 2, 8, 37, 512, 1024,
                       "64 frames x 256 tokens, SigLIP-shaped tower + 4-layer Qwen2.5-7B-shaped LLM, SP=2"),
        "c3": Workload("c3", c3, 256, 4, 8, 37, 512, 1024,
                       "256 frames x 256 tokens, 28-layer Qwen2.5-7B-shaped prefill, SP=4, G=8"),
        "c4": Workload("c4", c3, 512, 8, 8, 37, 512, 1024,
                       "512 frames x 256 tokens (~131K tokens), 7B-shaped encode+prefill, SP=8"),
        "c5": Workload("c5", c3, 1024, 8, 8, 37, 512, 1024,
                       "1024 frames (~262K tokens), 7B-shaped prefill, policy + reference, SP=8"),
    }


@dataclass
class Group:
    """A GRPO group's token data: question + G responses padded to Lmax."""
    question: np.ndarray  # int32 [n_q]
    resp: np.ndarray      # int32 [G, Lmax] (PAD past lengths)
    lengths: np.ndarray   # int32 [G]

    @property
    def Lmax(self) -> int:
        return int(self.resp.shape[1])

    @property
    def scored(self) -> int:
        return int(self.lengths.sum())


def make_group(w: Workload, seed: int = 3) -> Group:
    """Seeded synthetic group: content tokens U[kContentBase, V), lengths
    U[len_lo, len_hi] (SURVEY §8d value distributions)."""
    rng = np.random.default_rng(seed)
    V = w.cfg.vocab
    q = rng.integers(K_CONTENT_BASE, V, size=w.n_question, dtype=np.int64).astype(np.int32)
    lengths = rng.integers(w.len_lo, w.len_hi + 1, size=w.G).astype(np.int32)
    Lmax = int(lengths.max())
    resp = np.full((w.G, Lmax), K_PAD, dtype=np.int32)
    for g in range(w.G):
        resp[g, : lengths[g]] = rng.integers(K_CONTENT_BASE, V, size=int(lengths[g]))
    return Group(q, resp, lengths)


def gen_video(seed: int, frames: int, feature_dim: int) -> np.ndarray:
    """mmseq::gen_video as fp32 (mrsp_gen_video)."""
    out = np.empty((frames, feature_dim), dtype=np.float32)
    check(_lib.lib().mrsp_gen_video(seed, frames, feature_dim,
                                    out.ctypes.data_as(ctypes.POINTER(ctypes.c_float))))
    return out


def video_id(seed: int, frames: int) -> str:
    return f"v{seed}f{frames}"  # mmseq.cpp:64


def ulysses_plan(n_q: int, n_kv: int, sp: int, rank: int) -> dict:
    """Head split + all-to-all column blocks of one SP rank (mrsp_ulysses_plan)."""
    out = (ctypes.c_int32 * 14)()
    check(_lib.lib().mrsp_ulysses_plan(n_q, n_kv, sp, rank, out))
    v = list(out)
    return {"q": (v[0], v[1]), "kv": (v[2], v[3]), "q_per_kv": v[4],
            "blocks": [tuple(v[5 + 3 * i: 8 + 3 * i]) for i in range(3)]}


def head_split(n_q: int, n_kv: int, sp: int, rank: int, row_split: bool = True) -> dict:
    """The engine's head split of one SP rank (mrsp_head_split): query / kv head
    ranges and, above the kv-head count, the query-row split part."""
    out = (ctypes.c_int32 * 7)()
    check(_lib.lib().mrsp_head_split(n_q, n_kv, sp, rank, int(row_split), out))
    v = list(out)
    return {"q": (v[0], v[1]), "kv": (v[2], v[3]), "q_per_kv": v[4], "row_parts": v[5],
            "row_part": v[6]}


def attn_row_part(block: int, n_blocks: int, m: int) -> int:
    return int(_lib.lib().mrsp_attn_row_part(block, n_blocks, m))


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    check(_lib.lib().mrsp_nccl_unique_id(buf))
    return buf.raw


def _ptr(a, t=ctypes.c_int32):
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return ctypes.cast(ctypes.c_void_p(a.data_ptr()), ctypes.POINTER(t))
    return a.ctypes.data_as(ctypes.POINTER(t))


def _i32(a) -> np.ndarray:
    """Host int32 buffer the C side reads (a caller's int64 array would
    otherwise be reinterpreted)."""
    return np.ascontiguousarray(np.asarray(a), dtype=np.int32)


def _group_arrays(group: "Group"):
    q, resp, lens = _i32(group.question).reshape(-1), _i32(group.resp), _i32(group.lengths)
    if resp.ndim != 2 or lens.shape != (resp.shape[0],):
        raise ValueError(f"group: resp must be [G, Lmax] and lengths [G], got {resp.shape} / "
                         f"{lens.shape}")
    return q, resp, lens


def _pixels(pixels, cfg: "ModelConfig"):
    """(pointer, F, on_device) for a [F, 3*S*S] fp32 host array or CUDA tensor."""
    want = 3 * cfg.image_size ** 2
    if hasattr(pixels, "is_cuda"):
        import torch
        if not pixels.is_cuda or pixels.dtype != torch.float32 or not pixels.is_contiguous() \
                or pixels.dim() != 2 or pixels.shape[1] != want:
            raise ValueError(f"pixels: need a contiguous float32 CUDA tensor [F, {want}]")
        return _ptr(pixels, ctypes.c_float), int(pixels.shape[0]), 1, pixels
    arr = np.ascontiguousarray(pixels, dtype=np.float32)
    if arr.ndim != 2 or arr.shape[1] != want:
        raise ValueError(f"pixels: need [F, {want}] float32, got {arr.shape}")
    return _ptr(arr, ctypes.c_float), int(arr.shape[0]), 0, arr


def _out_tensor(t, n: int, name: str):
    import torch
    if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous() and t.numel() >= n):
        raise ValueError(f"{name}: need a contiguous float32 CUDA tensor with >= {n} elements")
    return t


class Engine:
    """One process's share of an SP group (sp virtual ranks when n_procs == 1)."""

    def __init__(self, cfg: ModelConfig, sp: int = 1, rank: int = 0, n_procs: int = 1,
                 vision_seed: int = 2, policy_seed: int = 3, ref_seed: int = 4,
                 with_ref: bool = True, nccl_id: Optional[bytes] = None):
        self.cfg = cfg
        self.sp = sp
        self._h = ctypes.c_void_p()
        idb = ctypes.create_string_buffer(nccl_id, 128) if nccl_id else None
        check(_lib.lib().mrsp_engine_create(ctypes.byref(cfg), sp, rank, n_procs, vision_seed,
                                            policy_seed, ref_seed, int(with_ref), idb,
                                            ctypes.byref(self._h)))

    # ---- rollout generation ------------------------------------------------
    def generate(self, vid: str, question, G: int, max_len: int, temperature: float = 1.0,
                 seed: int = 0):
        """Samples G rollouts after [cached video | question]; returns
        (tokens [G, max_len] int32, lengths [G], old_logprobs [G, max_len])."""
        q = np.ascontiguousarray(np.asarray(question, dtype=np.int32))
        tok = np.zeros((G, max_len), dtype=np.int32)
        lens = np.zeros(G, dtype=np.int32)
        olp = np.zeros((G, max_len), dtype=np.float32)
        check(_lib.lib().mrsp_engine_generate(self._h, vid.encode(), _ptr(q), len(q), G, max_len,
                                              float(temperature), int(seed), _ptr(tok), _ptr(lens),
                                              _ptr(olp, ctypes.c_float)))
        return tok, lens, olp

    # ---- weights (safetensors, HF names) -------------------------------------
    VISION, POLICY, REFERENCE = 0, 1, 2

    def save_weights(self, path: str) -> None:
        check(_lib.lib().mrsp_engine_save_weights(self._h, str(path).encode()))

    def load_weights(self, path: str, part: int, prefix: str = "") -> None:
        """part: Engine.VISION (tower + projector), POLICY or REFERENCE LLM, read
        from the tensors named `prefix` + the HF name."""
        check(_lib.lib().mrsp_engine_load_weights(self._h, str(path).encode(), part,
                                                  prefix.encode()))

    # ---- embedding-cache persistence ---------------------------------------
    def cache_save(self, vid: str, path: str) -> None:
        check(_lib.lib().mrsp_engine_cache_save(self._h, vid.encode(), str(path).encode()))

    def cache_load(self, vid: str, path: str) -> int:
        """Loads saved embeddings under `vid`; returns the frame count."""
        f = ctypes.c_int(0)
        check(_lib.lib().mrsp_engine_cache_load(self._h, vid.encode(), str(path).encode(),
                                                ctypes.byref(f)))
        return f.value

    # ---- peer-memory transport (one process per GPU, no NCCL) -------------
    def p2p_export(self, max_frames: int, max_tokens: int, max_scored: int) -> bytes:
        """Allocates this rank's IPC landing buffers; returns its blob for the
        host all-gather (engine created with n_procs > 1 and no nccl_id)."""
        n = _lib.lib().mrsp_p2p_blob_bytes()
        buf = ctypes.create_string_buffer(n)
        check(_lib.lib().mrsp_engine_p2p_export(self._h, max_frames, max_tokens, max_scored, buf))
        return buf.raw

    def p2p_import(self, blobs) -> None:
        """Maps every rank's landing buffers; blobs in rank order."""
        data = b"".join(blobs)
        check(_lib.lib().mrsp_engine_p2p_import(self._h, ctypes.create_string_buffer(data, len(data))))

    def close(self):
        if self._h:
            check(_lib.lib().mrsp_engine_destroy(self._h))
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return int(_lib.lib().mrsp_engine_stream(self._h) or 0)

    def encode(self, vid: str, pixels, use_cache: bool = True) -> bool:
        """Stage 1; pixels [F, 3*S*S] fp32 numpy (host) or torch CUDA tensor."""
        pp, F, on_dev, _keep = _pixels(pixels, self.cfg)
        hit = ctypes.c_int(0)
        check(_lib.lib().mrsp_engine_encode(self._h, vid.encode(), pp, F, on_dev, int(use_cache),
                                            ctypes.byref(hit)))
        return bool(hit.value)

    def prefill_logprobs(self, vid: str, group: Group, model: int = 0, with_lse: bool = False):
        q, resp, lens = _group_arrays(group)
        n = int(lens.sum())
        lp = np.zeros(n, dtype=np.float32)
        lse = np.zeros(n, dtype=np.float32) if with_lse else None
        check(_lib.lib().mrsp_engine_prefill_logprobs(
            self._h, vid.encode(), _ptr(q), len(q), _ptr(resp), _ptr(lens), int(resp.shape[0]),
            int(resp.shape[1]), model, _ptr(lp, ctypes.c_float), _ptr(lse, ctypes.c_float), 0))
        return (lp, lse) if with_lse else lp

    def step(self, vid: str, pixels, group: Group, use_cache: bool = True, out=None,
             with_kl: bool = False):
        """run_step: G fetches + policy and reference log-probs (+ exact per-token
        KL from the fused dual LM head). `out` = optional tuple of device tensors
        (lp_policy, lp_ref[, kl]) to receive the results without a D2H copy."""
        pp, F, on_dev, _keep = _pixels(pixels, self.cfg)
        q, resp, lens = _group_arrays(group)
        n = int(lens.sum())
        if out is None:
            lp_p = np.zeros(n, dtype=np.float32)
            lp_r = np.zeros(n, dtype=np.float32)
            kl = np.zeros(n, dtype=np.float32) if with_kl else None
            out_dev = 0
        else:
            lp_p = _out_tensor(out[0], n, "out[0]")
            lp_r = _out_tensor(out[1], n, "out[1]")
            kl = _out_tensor(out[2], n, "out[2]") if len(out) > 2 else None
            out_dev = 1
        check(_lib.lib().mrsp_engine_step(
            self._h, vid.encode(), pp, F, on_dev, int(use_cache), _ptr(q), len(q), _ptr(resp),
            _ptr(lens), int(resp.shape[0]), int(resp.shape[1]), _ptr(lp_p, ctypes.c_float),
            _ptr(lp_r, ctypes.c_float), _ptr(kl, ctypes.c_float), out_dev))
        return (lp_p, lp_r, kl) if with_kl or (out is not None and len(out) > 2) else (lp_p, lp_r)

    # ---- GRPO backward -----------------------------------
    def grpo_backward(self, vid: str, group: Group, old_logprobs, advantages,
                      clip_eps: float = 0.2, kl_beta: float = 0.04, sampled_kl: bool = False):
        """grpo_gradient (grpo.cpp:122-206) through the transformer-shaped prefill:
        the policy LLM's fp32 gradients stay in the engine (save_grads). Returns
        (stats {objective, mean_kl, clip_fraction, token_count}, policy log-probs)."""
        q, resp, lens = _group_arrays(group)
        n = int(lens.sum())
        old = np.ascontiguousarray(old_logprobs, dtype=np.float32).reshape(-1)
        adv = np.ascontiguousarray(advantages, dtype=np.float32).reshape(-1)
        if old.shape != (n,) or adv.shape != (resp.shape[0],):
            raise ValueError(f"grpo_backward: old_logprobs needs {n} and advantages "
                             f"{resp.shape[0]} entries")
        st = np.zeros(4, dtype=np.float64)
        lp = np.zeros(n, dtype=np.float32)
        check(_lib.lib().mrsp_engine_grpo_backward(
            self._h, vid.encode(), _ptr(q), len(q), _ptr(resp), _ptr(lens), int(resp.shape[0]),
            int(resp.shape[1]), _ptr(old, ctypes.c_float), _ptr(adv, ctypes.c_float),
            float(clip_eps), float(kl_beta), int(sampled_kl), _ptr(st, ctypes.c_double),
            _ptr(lp, ctypes.c_float)))
        return dict(zip(["objective", "mean_kl", "clip_fraction", "token_count"],
                        [float(x) for x in st])), lp

    def sft_backward(self, vid: str, group: Group):
        """sft_loss_and_grad (grpo.cpp:208-223) over the group's rows as
        teacher-forced targets; returns (loss, policy log-probs); gradients of
        the loss stay in the engine (save_grads)."""
        q, resp, lens = _group_arrays(group)
        lp = np.zeros(int(lens.sum()), dtype=np.float32)
        loss = ctypes.c_double()
        check(_lib.lib().mrsp_engine_sft_backward(
            self._h, vid.encode(), _ptr(q), len(q), _ptr(resp), _ptr(lens), int(resp.shape[0]),
            int(resp.shape[1]), ctypes.byref(loss), _ptr(lp, ctypes.c_float)))
        return float(loss.value), lp

    def save_grads(self, path: str) -> None:
        check(_lib.lib().mrsp_engine_save_grads(self._h, str(path).encode()))

    def stats(self, reset: bool = False) -> dict:
        out = (ctypes.c_uint64 * 6)()
        check(_lib.lib().mrsp_engine_stats(self._h, out, int(reset)))
        return dict(zip(["encoder_invocations", "cache_hits", "cache_misses", "gather_bytes",
                         "pad_reads", "a2a_bytes"], [int(x) for x in out]))

    def cache_size(self) -> int:
        n = ctypes.c_uint64()
        check(_lib.lib().mrsp_engine_cache(self._h, 0, 0, ctypes.byref(n)))
        return int(n.value)

    def cache_clear(self):
        check(_lib.lib().mrsp_engine_cache(self._h, 1, 0, None))

    def cache_capacity(self, n: int):
        check(_lib.lib().mrsp_engine_cache(self._h, 2, n, None))

    def embedding_frames(self, vid: str) -> int:
        f = ctypes.c_int(0)
        check(_lib.lib().mrsp_engine_get_embeddings(self._h, vid.encode(), None, 0,
                                                    ctypes.byref(f)))
        return f.value

    def embeddings(self, vid: str, frames: Optional[int] = None) -> np.ndarray:
        """Cached [F*T, dim] embeddings as float32 (from bf16). The buffer is
        sized from the entry (frames, when given, must match it)."""
        T = self.cfg.tokens_per_frame
        F = self.embedding_frames(vid)
        if frames is not None and frames != F:
            raise ValueError(f"embeddings: {vid} holds {F} frames, not {frames}")
        raw = np.empty((F * T, self.cfg.dim), dtype=np.uint16)
        check(_lib.lib().mrsp_engine_get_embeddings(self._h, vid.encode(),
                                                    raw.ctypes.data_as(ctypes.c_void_p),
                                                    raw.nbytes, None))
        return (raw.astype(np.uint32) << 16).view(np.float32)

    PROFILE_CLASSES = ["llm_attention", "llm_gemm", "vision", "lm_head", "collectives", "misc",
                       "decode_graph", "backward", "attention_backward"]

    def profile(self, enable: Optional[bool] = None) -> dict:
        en = -1 if enable is None else int(enable)
        check(_lib.lib().mrsp_engine_profile(self._h, en, 0, None, None))
        out = {}
        for i, name in enumerate(self.PROFILE_CLASSES):
            ms = ctypes.c_double()
            n = ctypes.c_int64()
            check(_lib.lib().mrsp_engine_profile(self._h, -1, i, ctypes.byref(ms), ctypes.byref(n)))
            out[name] = (ms.value, n.value)
        return out


def read_safetensors(path: str) -> dict:
    """{name: float32 numpy array} from a safetensors file (F32 / BF16 tensors;
    the engine's weights and gradients), without the safetensors package."""
    import json
    import struct
    with open(path, "rb") as f:
        n = struct.unpack("<Q", f.read(8))[0]
        hdr = json.loads(f.read(n))
        data = f.read()
    out = {}
    for name, t in hdr.items():
        if name == "__metadata__":
            continue
        b, e = t["data_offsets"]
        raw = np.frombuffer(data[b:e], dtype=np.uint16 if t["dtype"] == "BF16" else np.float32)
        if t["dtype"] == "BF16":
            raw = (raw.astype(np.uint32) << 16).view(np.float32)
        out[name] = raw.reshape(t["shape"])
    return out
