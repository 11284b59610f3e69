"""GPU: the reference's toy MR-SP path on the device (csrc/toy.cu) through the
C-ABI, bit-exact against the reference's own outputs (golden fixture) and the
CPU oracle; the reference's unmodified unit tests + acceptance C4/C5 linked
against the B200 engine in place of src/engine.cpp."""
import json
import os
import pathlib
import subprocess
import threading

import numpy as np
import pytest

from oracle import toy
from paper_2507_07966_b200 import mrsp

pytestmark = pytest.mark.gpu
ROOT = pathlib.Path(__file__).resolve().parents[1]
GOLD = json.loads((ROOT / "tests" / "golden" / "ref_toy.json").read_text())


def enc_params(seed, d, p):
    return mrsp.EncoderParams(d, p, toy.encoder_generate(seed, d, p))


def test_encode_golden_bit_exact(gpu):
    enc = enc_params(1234, 8, 16)
    got = mrsp.serial_encode(enc, toy.gen_video(9, 5, 16))
    assert got.tolist() == GOLD["encode_v9f5"]
    encb = enc_params(1234, 128, 256)
    got = mrsp.serial_encode(encb, toy.gen_video(1234 + 64 * 100, 3, 256))
    assert got.tolist() == GOLD["encode_bench_shape"]


def test_parallel_encode_matches_oracle_all_sp(gpu):
    # test_engine.cpp:57-70 and acceptance C4 shape, vs the CPU oracle.
    enc = enc_params(3, 16, 32)
    for seed in range(25):
        frames = toy.gen_video(seed, 3 + seed % 9, 32)
        want = toy.serial_encode(enc.w, frames)
        for sp in (1, 2, 3, 4, 8):
            g = mrsp.WorkerGroup(sp, enc)
            plan = mrsp.plan_shards(frames.shape[0], sp)
            got = mrsp.all_gather(g.parallel_encode(frames, plan), sp, None)
            assert np.array_equal(got, want)
            assert g.stats().encoder_invocations == frames.shape[0]


def test_bench_shape_encode_512_frames(gpu):
    enc = enc_params(1234, 128, 256)
    frames = toy.gen_video(1234 + 512 * 100, 512, 256)
    want = toy.serial_encode(enc.w, frames)
    g = mrsp.WorkerGroup(8, enc)
    got = mrsp.all_gather(g.parallel_encode(frames, mrsp.plan_shards(512, 8)), 8, g.stats())
    assert np.array_equal(got, want)
    assert g.stats().gather_bytes == 512 * 128 * 7 * 8


def test_prefill_golden_bit_exact(gpu):
    theta = np.array(GOLD["policy_32_8_12_seed4"])
    params = mrsp.PolicyParams(32, 8, 12, theta)
    pf = GOLD["prefill"]
    batch = mrsp.pad_batch(pf["rows"])
    for sp in (1, 2, 3, 4):
        g = mrsp.WorkerGroup(sp, enc_params(3, 8, 16))
        out = g.parallel_prefill(params, np.array(pf["contexts"]), batch,
                                 mrsp.plan_shards(batch.max_len, sp))
        assert [o.tolist() for o in out] == pf["logits"]
        assert g.stats().pad_reads == 0


def test_prefill_random_batches_vs_oracle(gpu):
    # test_engine.cpp:155-187 (50 trials, sp 1-4) against the CPU oracle.
    V, d, h = 32, 8, 12
    theta = toy.policy_random(V, d, h, 4, 0.4)
    params = mrsp.PolicyParams(V, d, h, theta)
    rng = np.random.default_rng(31)
    for trial in range(50):
        n_rows = int(rng.integers(1, 7))
        rows = [rng.integers(1, 32, size=int(rng.integers(1, 10))).tolist() for _ in range(n_rows)]
        ctx = rng.standard_normal((n_rows, d))
        batch = mrsp.pad_batch(rows)
        want = toy.serial_prefill(theta, V, d, h, ctx, batch.rows, batch.lengths)
        sp = 1 + trial % 4
        g = mrsp.WorkerGroup(sp, enc_params(3, 8, 16))
        got = g.parallel_prefill(params, ctx, batch, mrsp.plan_shards(batch.max_len, sp))
        assert np.array_equal(np.concatenate(got), want)
        assert g.stats().pad_reads == 0


def test_prefill_errors(gpu):
    params = mrsp.PolicyParams(32, 8, 12, toy.policy_random(32, 8, 12, 4, 0.4))
    batch = mrsp.pad_batch([[40]])  # token out of range -> step_logits error at t=1? len 1 -> prev EOS
    g = mrsp.WorkerGroup(1, enc_params(3, 8, 16))
    g.parallel_prefill(params, np.zeros((1, 8)), batch, mrsp.plan_shards(1, 1))
    bad = mrsp.pad_batch([[40, 5]])
    with pytest.raises(mrsp.InvalidArgument, match="prev token out of range"):
        g.parallel_prefill(params, np.zeros((1, 8)), bad, mrsp.plan_shards(2, 1))
    with pytest.raises(mrsp.InvalidArgument, match="does not cover the padded length"):
        g.parallel_prefill(params, np.zeros((1, 8)), bad, mrsp.plan_shards(3, 1))


def test_cache_exactly_once_concurrent(gpu):
    # test_engine.cpp:223-241
    enc = enc_params(8, 8, 16)
    frames = toy.gen_video(3, 10, 16)
    plan = mrsp.plan_shards(10, 1)
    for _ in range(5):
        g = mrsp.WorkerGroup(1, enc)
        cache = mrsp.EmbeddingCache()
        res = [None] * 8
        th = [threading.Thread(target=lambda t=t: res.__setitem__(
            t, cache.get_or_encode(g, "v3f10", frames, plan)[0])) for t in range(8)]
        [t.start() for t in th]
        [t.join() for t in th]
        assert g.stats().encoder_invocations == 10
        assert g.stats().cache_misses == 1 and g.stats().cache_hits == 7
        assert all(r is res[0] for r in res)


REF_BINS = ["test_engine", "test_policy", "test_grpo", "test_mmseq"]


@pytest.mark.parametrize("name", REF_BINS)
def test_reference_unit_tests_against_b200_engine(gpu, name):
    exe = ROOT / "oracle" / "_ref" / "dropin" / name
    if not exe.exists():
        pytest.skip(f"{exe} not built (needs /root/reference at build time)")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "0 failed" in r.stdout


def test_reference_acceptance_c4_c5_against_b200_engine(gpu):
    exe = ROOT / "oracle" / "_ref" / "dropin" / "acceptance"
    if not exe.exists():
        pytest.skip("acceptance drop-in not built")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=900,
                       env={**os.environ, "LVRL_BIN": "/nonexistent"})
    lines = [l for l in r.stdout.splitlines() if l.startswith("criterion")]
    got = {l.split(":")[0]: l for l in lines}
    for c in ("criterion 1", "criterion 2", "criterion 3", "criterion 4", "criterion 5"):
        assert c in got and "PASS" in got[c], r.stdout[-4000:] + r.stderr[-2000:]
