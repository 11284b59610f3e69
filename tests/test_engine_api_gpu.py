"""GPU: engine C-ABI contract checks — concurrent exactly-once fetches through
Engine::get_or_encode (test_engine.cpp:223-241 on the device engine), argument
validation of the step entry point and the embeddings copy-out capacity."""
import threading

import numpy as np
import pytest

from paper_2507_07966_b200 import _lib, engine as E

pytestmark = pytest.mark.gpu

W1 = E.workloads()["c1"]


def test_concurrent_encode_exactly_once(gpu):
    """8 host threads fetch the same video through mrsp_engine_encode: one
    miss fills the entry (F encoder invocations), the other 7 hit, and all
    see the same embeddings (the reference's 8-concurrent-callers KAT)."""
    eng = E.Engine(W1.cfg, sp=2, vision_seed=2, policy_seed=3, ref_seed=4)
    pix = E.gen_video(1, W1.frames, 3 * W1.cfg.image_size ** 2)
    hits, errs = [], []
    start = threading.Barrier(8)

    def fetch():
        try:
            start.wait()
            hits.append(eng.encode("shared", pix))
        except Exception as ex:  # surfaced below
            errs.append(repr(ex))

    ts = [threading.Thread(target=fetch) for _ in range(8)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    st = eng.stats()
    assert sorted(hits) == [False] + [True] * 7
    assert st["cache_misses"] == 1 and st["cache_hits"] == 7
    assert st["encoder_invocations"] == W1.frames
    assert eng.cache_size() == 1
    ref = E.Engine(W1.cfg, sp=1, vision_seed=2, policy_seed=3, ref_seed=4)
    ref.encode("shared", pix)
    assert np.array_equal(eng.embeddings("shared"), ref.embeddings("shared"))
    ref.close()
    eng.close()


def test_step_rejects_empty_group_and_small_buffers(gpu):
    import ctypes
    eng = E.Engine(W1.cfg, sp=1, vision_seed=2, policy_seed=3, ref_seed=4)
    pix = E.gen_video(1, W1.frames, 3 * W1.cfg.image_size ** 2)
    eng.encode("v", pix)
    empty = E.Group(np.array([10], np.int32), np.zeros((0, 4), np.int32), np.zeros(0, np.int32))
    with pytest.raises(_lib.InvalidArgument):
        eng.step("v", pix, empty)
    with pytest.raises(_lib.InvalidArgument):
        eng.prefill_logprobs("v", empty)
    # embeddings copy-out: a short host buffer is refused, nothing written
    T = W1.cfg.tokens_per_frame
    assert eng.embedding_frames("v") == W1.frames
    small = np.full(((W1.frames - 1) * T, W1.cfg.dim), 7, dtype=np.uint16)
    with pytest.raises(_lib.InvalidArgument):
        _lib.check(_lib.lib().mrsp_engine_get_embeddings(
            eng._h, b"v", small.ctypes.data_as(ctypes.c_void_p), small.nbytes, None))
    assert (small == 7).all()
    with pytest.raises(ValueError):
        eng.embeddings("v", W1.frames - 1)
    eng.close()
