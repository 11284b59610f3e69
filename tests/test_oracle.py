"""CPU: pin the oracle (oracle/mrsp_oracle.c) to the reference's own outputs.

tests/golden/ref_toy.json was produced by oracle/gen_golden.cpp linked against
the reference sources (/root/reference/proj/src), see oracle/Makefile.
The survey's extra known-answer values are checked as well.
"""
import json
import pathlib
import subprocess

import numpy as np
import pytest

from oracle import toy

GOLD = json.loads((pathlib.Path(__file__).parent / "golden" / "ref_toy.json").read_text())


def test_plan_shards_golden():
    for case in GOLD["plan_shards"]:
        assert toy.plan_shards(case["n"], case["k"]) == [tuple(r) for r in case["ranges"]]


def test_plan_shards_lawful_partition():
    # test_engine.cpp:37-55
    for n in range(41):
        for k in range(1, n + 5):
            r = toy.plan_shards(n, k)
            assert len(r) == k and r[0][0] == 0 and r[-1][1] == n
            sizes = [e - b for b, e in r]
            assert max(sizes) - min(sizes) <= 1
            assert all(r[i][1] == r[i + 1][0] for i in range(k - 1))
    with pytest.raises(ValueError):
        toy.plan_shards(4, 0)


def test_survey_kats():
    assert int(toy.substream_draws(7, "video", 1)[0]) == 10773524323035910004
    assert str(int(toy.substream_draws(7, "video", 1)[0])) == GOLD["substream_7_video_first"]
    v = toy.gen_video(7, 2, 4)
    assert v.tolist() == GOLD["gen_video_7_2_4"]["frames"]
    assert toy.video_id(7, 2) == GOLD["gen_video_7_2_4"]["id"] == "v7f2"
    w = toy.encoder_generate(1234, 8, 16)
    assert w.reshape(-1)[64:67].tolist() == [0.32938537127381601, 0.34926642573245475,
                                            -0.26112000355548221]
    assert toy.plan_shards(131104, 8) == [(i * 16388, (i + 1) * 16388) for i in range(8)]


def test_encoder_and_encode_golden():
    w = toy.encoder_generate(1234, 8, 16)
    assert w.reshape(-1).tolist() == GOLD["encoder_1234_8_16"]
    frames = toy.gen_video(9, 5, 16)
    assert toy.serial_encode(w, frames).tolist() == GOLD["encode_v9f5"]
    wb = toy.encoder_generate(1234, 128, 256)
    fb = toy.gen_video(1234 + 64 * 100, 3, 256)
    assert toy.serial_encode(wb, fb).tolist() == GOLD["encode_bench_shape"]


def test_policy_step_logits_prefill_golden():
    theta = toy.policy_random(32, 8, 12, 4, 0.4)
    assert theta.tolist() == GOLD["policy_32_8_12_seed4"]
    logits = toy.step_logits(theta, 32, 8, 12, np.full(8, 0.1), 1)
    assert logits.tolist() == GOLD["step_logits_ctx01_eos"]
    assert toy.log_softmax(logits).tolist() == GOLD["log_softmax_of_that"]
    pf = GOLD["prefill"]
    rows = pf["rows"]
    L = max(len(r) for r in rows)
    padded = np.zeros((len(rows), L), dtype=np.int32)
    for i, r in enumerate(rows):
        padded[i, : len(r)] = r
    out = toy.serial_prefill(theta, 32, 8, 12, np.array(pf["contexts"]), padded,
                             np.array([len(r) for r in rows], dtype=np.uint64))
    want = [x for r in pf["logits"] for x in r]
    assert out.tolist() == want


def test_context_vector_golden():
    theta = toy.policy_random(32, 8, 12, 4, 0.4)
    emb = toy.serial_encode(toy.encoder_generate(2, 8, 16), toy.gen_video(3, 4, 16))
    assert toy.context_vector(theta, 32, 8, emb, [10, 11, 12]).tolist() == GOLD["context_vector"]


def test_glibc_tanh_model():
    """The device tanh (csrc/glibc_tanh.cuh) restates glibc's algorithm; this
    checks the same restatement, compiled for the host, against libm."""
    src = pathlib.Path(__file__).parent / "support" / "tanh_model.c"
    exe = pathlib.Path("/tmp/mrsp_tanh_model")
    subprocess.run(["/usr/bin/gcc", "-O2", "-mfma", "-ffp-contract=off", str(src), "-o", str(exe),
                    "-lm"], check=True)
    r = subprocess.run([str(exe), "2000000"], check=True, capture_output=True, text=True)
    assert r.stdout.strip().endswith("mismatches 0"), r.stdout


def test_grpo_stats_oracle_vs_reference():
    """oracle/grpo.py reproduces the reference's GroupStats (grpo_objective)."""
    from oracle import grpo
    g = GOLD["grpo"]
    r = g["rollouts"]
    for key, sampled in (("stats_exact_kl", False), ("stats_sampled_kl", True)):
        got = grpo.group_stats([x["logprobs"] for x in r], [x["old_logprobs"] for x in r],
                               [x["ref_logprobs"] for x in r], [x["kl"] for x in r],
                               g["advantages"], g["clip_eps"], g["kl_beta"], sampled)
        want = g[key]
        assert got["token_count"] == want["token_count"]
        assert got["clip_fraction"] == want["clip_fraction"]
        assert abs(got["objective"] - want["objective"]) < 1e-12
        assert abs(got["mean_kl"] - want["mean_kl"]) < 1e-12
