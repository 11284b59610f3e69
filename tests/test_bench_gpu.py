"""GPU: `bench.py --gpus 2` launches its own ranks (no external torchrun) and
reports one line for the whole job. MRSP_BENCH_SAME_DEVICE=1 puts both ranks
on device 0 (CUDA-IPC mappings of one GPU stand in for NVLink peers), so the
multi-process flow — peer-memory Ulysses exchanges, the video gather, the
per-rank timing and max-over-ranks — runs on a one-GPU box."""
import json
import os
import pathlib
import subprocess
import sys

import pytest

from paper_2507_07966_b200 import engine as E

pytestmark = pytest.mark.gpu
ROOT = pathlib.Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("comm", ["p2p", "nccl"])
def test_bench_self_launches_two_ranks(gpu, comm):
    """comm "nccl": the NCCL transport (MRSP_COMM=nccl), the two ranks on
    separate NCCL host ids (its socket transport; tests/test_nccl_gpu.py)."""
    env = {**os.environ, "MRSP_BENCH_SAME_DEVICE": "1", "MRSP_COMM": comm}
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--workload", "c1",
                          "--steps", "1", "--warmup", "3", "--no-cpu", "--no-gen"],
                         capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-4000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 only
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["config"]["sp_degree"] == 2
    assert "comm" not in line["config"]
    c = line["counters_per_step"]
    w = E.workloads()["c1"]
    T = w.cfg.tokens_per_frame
    # the reference's all_gather accounting (engine.cpp:149-151): values x
    # (sp - 1) x bytes per value, here bf16 values of the gathered video
    assert c["a2a_bytes"] > 0
    assert c["gather_bytes"] == w.frames * T * w.cfg.dim * (2 - 1) * 2
    assert c["encoder_invocations"] == w.frames // 2  # rank 0's shard: plan_shards(8, 2)
    assert [r["rank"] for r in line["kernel_ms_per_rank"]] == [0, 1]
    assert line["value"] > 0 and line["gpu_launches"] > 0
