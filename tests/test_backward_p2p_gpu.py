"""GPU: the GRPO backward across PROCESSES (one process per GPU over the CUDA-IPC
peer mesh, no NCCL), run as 2 processes sharing one B200 (IPC mappings of one
device stand in for NVLink peers): the recompute's fused QKV scatter into the
peers' head shards, O / dO / dq-dk-dv exchanged between sequence and head
shards through the mesh's landing buffers, the LM-head slices' dX rows to the
token owners, and the weight gradients summed across ranks in rank order
through the staging slots. Every rank must hold the same gradients, equal to
the one-process SP engine's (virtual ranks: same per-token arithmetic, same
rank-order sums), and the group statistics must equal SP = 1's."""
import multiprocessing as mp
import os
import socket
import tempfile

import numpy as np
import pytest

from paper_2507_07966_b200 import engine as E

pytestmark = pytest.mark.gpu

W1 = E.workloads()["c1"]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs():
    pix = E.gen_video(1, W1.frames, 3 * W1.cfg.image_size ** 2)
    grp = E.make_group(W1, seed=6)
    n = grp.scored
    rng = np.random.default_rng(2)
    old = (-3.5 + rng.normal(0, 0.2, size=n)).astype(np.float32)
    adv = rng.normal(size=W1.G).astype(np.float32)
    return pix, grp, old, adv


def _worker(rank, world, port, q, td):
    try:
        import torch
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        pix, grp, old, adv = _inputs()
        eng = E.Engine(W1.cfg, sp=world, rank=rank, n_procs=world, vision_seed=2,
                       policy_seed=3, ref_seed=4)
        L = W1.frames * W1.cfg.tokens_per_frame + len(grp.question) + grp.resp.shape[0] * grp.Lmax
        blob = eng.p2p_export(W1.frames, L, grp.scored)
        blobs = [None] * world
        dist.all_gather_object(blobs, blob)
        eng.p2p_import(blobs)
        eng.encode("v", pix)
        out = []
        for i in range(2):  # a second call reuses every landing buffer
            st, lp = eng.grpo_backward("v", grp, old, adv)
            path = os.path.join(td, f"g{rank}_{i}.safetensors")
            eng.save_grads(path)
            out.append((st, lp, path))
        lp_p, _ = eng.step("v", pix, grp)  # the forward still works after the backward
        dist.barrier()
        eng.close()
        dist.destroy_process_group()
        q.put((rank, out, lp_p, None))
    except Exception as ex:  # surfaced by the parent
        q.put((rank, None, None, repr(ex)))


@pytest.mark.parametrize("world", [2, 4])
def test_grpo_backward_processes_match_virtual_ranks(gpu, world):
    """world 4 > 2 kv heads: the query-row split, each kv head's dK / dV
    partials summed on the token owners."""
    pix, grp, old, adv = _inputs()
    with tempfile.TemporaryDirectory() as td:
        ref = {}
        for sp in (1, world):
            eng = E.Engine(W1.cfg, sp=sp, vision_seed=2, policy_seed=3, ref_seed=4)
            eng.encode("v", pix)
            st, lp = eng.grpo_backward("v", grp, old, adv)
            path = os.path.join(td, f"virt{sp}.safetensors")
            eng.save_grads(path)
            lp_fwd, _ = eng.step("v", pix, grp)
            eng.close()
            ref[sp] = (st, lp, E.read_safetensors(path), lp_fwd)
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        port = _free_port()
        procs = [ctx.Process(target=_worker, args=(r, world, port, q, td)) for r in range(world)]
        for p in procs:
            p.start()
        res = sorted([q.get(timeout=900) for _ in range(world)], key=lambda r: r[0])
        for p in procs:
            p.join(timeout=120)
        for rank, out, lp_p, err in res:
            assert err is None, (rank, err)
            assert np.array_equal(lp_p, ref[1][3]), rank
            for st, lp, path in out:
                assert np.array_equal(lp, ref[1][1]), rank
                assert st == ref[1][0], rank
                got = E.read_safetensors(path)
                want = ref[world][2]
                for name in want:
                    assert np.array_equal(got[name], want[name]), (rank, name)
