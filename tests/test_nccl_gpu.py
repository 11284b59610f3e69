"""GPU: the NCCL transport of the one-process-per-GPU engine (MRSP_COMM=nccl in
bench.py; csrc/comm.cpp + the nccl_ branches of csrc/engine.cu) — Stage 1's
ncclAllGather of the projector output, Stage 2's grouped ncclSend / ncclRecv
all-to-alls per layer and the log-prob ncclAllReduce — run as 2 and 4 processes
sharing one B200.

NCCL refuses two ranks of one communicator on the same GPU of the same host, so
each process gets its own NCCL_HOSTID: NCCL then treats the ranks as separate
hosts and moves the data over its socket transport on the loopback interface.
That exercises every NCCL call, buffer size and per-peer offset of the data
plane on the hardware (not the NVLink bandwidth). Every rank's outputs must be
bit-identical to the single-process SP = 1 engine, as for the peer-memory path
(tests/test_p2p_gpu.py)."""
import multiprocessing as mp
import os
import queue
import socket

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
    grp = E.make_group(W1, seed=3)
    return pix, grp


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                          NCCL_HOSTID=f"mrsp-nccl-test-{rank}", NCCL_SOCKET_IFNAME="lo",
                          NCCL_IB_DISABLE="1")
        import torch
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        obj = [E.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        pix, grp = _inputs()
        eng = E.Engine(W1.cfg, sp=world, rank=rank, n_procs=world, vision_seed=2,
                       policy_seed=3, ref_seed=4, nccl_id=obj[0])
        out = []
        for i in range(2):  # a second video + step reuses the transport buffers
            eng.encode(f"v{i}", pix)
            out.append(eng.step(f"v{i}", pix, grp, with_kl=True))
        emb = eng.embeddings("v0", W1.frames)
        st = eng.stats()
        dist.barrier()
        eng.close()
        dist.destroy_process_group()
        q.put((rank, out, emb, st, None))
    except Exception as ex:  # surfaced by the parent
        q.put((rank, None, None, None, repr(ex)))


def _run(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = []
    try:
        for _ in range(world):
            res.append(q.get(timeout=420))
    except queue.Empty:
        pass
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    assert len(res) == world, f"only {len(res)} of {world} ranks finished (NCCL hang?)"
    return sorted(res, key=lambda r: r[0])


@pytest.mark.parametrize("world", [2, 4])
def test_nccl_processes_bit_exact_vs_sp1(gpu, world):
    pix, grp = _inputs()
    base = E.Engine(W1.cfg, sp=1, vision_seed=2, policy_seed=3, ref_seed=4)
    base.encode("v0", pix)
    want = base.step("v0", pix, grp, with_kl=True)
    want_emb = base.embeddings("v0", W1.frames)
    base.close()
    res = _run(world)
    for rank, out, emb, st, err in res:
        assert err is None, f"rank {rank}: {err}"
        assert np.array_equal(emb, want_emb), f"rank {rank}: gathered video embeddings differ"
        for lp_p, lp_r, kl in out:
            assert np.array_equal(lp_p, want[0]), f"rank {rank}: policy log-probs differ"
            assert np.array_equal(lp_r, want[1]), f"rank {rank}: reference log-probs differ"
            assert np.array_equal(kl, want[2]), f"rank {rank}: KL differs"
        T = W1.cfg.tokens_per_frame
        assert st["gather_bytes"] == 2 * W1.frames * T * W1.cfg.dim * (world - 1) * 2
        assert st["a2a_bytes"] > 0 and st["cache_misses"] == 2
