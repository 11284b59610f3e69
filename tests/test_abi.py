"""CPU: the C-ABI library loads and exports every symbol include/*.h declares;
host-only entry points work without a GPU; compute entry points fail loudly
(no CPU fallback)."""
import pathlib
import re

import numpy as np
import pytest

from paper_2507_07966_b200 import _lib, mrsp

ROOT = pathlib.Path(__file__).resolve().parents[1]


def declared_symbols():
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        names |= set(re.findall(r"\b(mrsp_[a-z0-9_]+)\s*\(", text))
    return sorted(names)


def test_every_declared_symbol_is_exported():
    lib = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 5
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_every_declared_symbol_has_a_ctypes_signature():
    _lib.lib()
    missing = [s for s in declared_symbols() if s not in _lib.SIGNATURES]
    assert not missing, missing


def test_version_and_plan_without_gpu():
    assert b"sm_100a" in _lib.lib().mrsp_version()
    p = mrsp.plan_shards(10, 3)
    assert p.ranges == [(0, 4), (4, 7), (7, 10)] and p.total == 10
    assert mrsp.plan_shards(2, 4).ranges == [(0, 1), (1, 2), (2, 2), (2, 2)]
    with pytest.raises(mrsp.InvalidArgument, match="sp_degree must be >= 1"):
        mrsp.plan_shards(4, 0)


def test_pad_batch_host_logic():
    b = mrsp.pad_batch([[5, 6, 7], [8], [9, 10, 11, 12, 13], []])
    assert b.max_len == 5 and b.rows.shape == (4, 5)
    assert mrsp.unpad_batch(b) == [[5, 6, 7], [8], [9, 10, 11, 12, 13], []]
    assert (b.rows[1, 1:] == mrsp.K_PAD).all()
    with pytest.raises(mrsp.InvalidArgument):
        mrsp.pad_batch([])


def test_all_gather_host_logic():
    sl = [mrsp.EncodedSlice(1, 2, 4, np.ones((2, 3))), mrsp.EncodedSlice(0, 0, 2, np.zeros((2, 3)))]
    st = mrsp.EngineStats()
    out = mrsp.all_gather(sl, 2, st)
    assert out.shape == (4, 3) and (out[:2] == 0).all() and st.gather_bytes == 12 * 1 * 8
    with pytest.raises(mrsp.GatherError):
        mrsp.all_gather(sl[:1], 2, None)
    with pytest.raises(mrsp.GatherError):
        mrsp.all_gather([], 2, None)


def test_compute_fails_loudly_without_gpu():
    if _lib.device_count() > 0:
        pytest.skip("a GPU is visible")
    enc = mrsp.EncoderParams(4, 8, np.ones((4, 8)))
    with pytest.raises(_lib.MrspError, match="no CPU fallback"):
        mrsp.serial_encode(enc, np.ones((2, 8)))


def test_gen_video_matches_reference_golden():
    """mrsp_gen_video (the engine's frame source) is float32 of the reference's
    fp64 gen_video(7, 2, 4) (mmseq.cpp:58-72), element for element."""
    import json
    from paper_2507_07966_b200 import engine as E
    gold = json.loads((ROOT / "tests" / "golden" / "ref_toy.json").read_text())["gen_video_7_2_4"]
    got = E.gen_video(7, 2, 4)
    assert got.dtype == np.float32
    assert np.array_equal(got, np.asarray(gold["frames"], dtype=np.float64).astype(np.float32))
    assert E.video_id(7, 2) == gold["id"]


def test_engine_front_end_validates_host_buffers():
    """The Python front-end coerces token arrays to int32 (a default-int64
    array must not be reinterpreted) and rejects mis-shaped pixels before any
    pointer reaches the C side."""
    from paper_2507_07966_b200 import engine as E
    w = E.workloads()["c1"]
    g = E.Group(np.array([10, 11], dtype=np.int64), np.array([[12, 13, 0], [14, 15, 16]]),
                np.array([2, 3]))
    q, resp, lens = E._group_arrays(g)
    assert q.dtype == resp.dtype == lens.dtype == np.int32
    assert lens.tolist() == [2, 3] and resp[1].tolist() == [14, 15, 16]
    with pytest.raises(ValueError):
        E._group_arrays(E.Group(q, resp, np.array([2, 3, 4])))
    with pytest.raises(ValueError):
        E._pixels(np.zeros((2, 10), np.float32), w.cfg)
    ptr, F, on_dev, keep = E._pixels(np.zeros((3, 3 * 64 * 64), np.float64), w.cfg)
    assert F == 3 and on_dev == 0 and keep.dtype == np.float32
