"""CPU, multi-process (gloo): the SP host logic of the NCCL path.

Each process is one SP rank. Using the library's own plans — plan_shards
(token shards, engine.cpp:15-29) and mrsp_ulysses_plan (head split + the
per-peer column blocks the engine's all-to-all sends) — the ranks exchange a
QKV activation sequence-shard -> head-shard with send/recv exactly as
Engine::a2a_forward does over NCCL, run attention on their heads (oracle
math), exchange back (a2a_backward), and must reproduce the single-rank result;
the Stage-1 frame plan + padded all-gather compaction is checked the same way.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import transformer as T
from paper_2507_07966_b200 import engine as E
from paper_2507_07966_b200 import mrsp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, nq, nkv, L, Lp, Lmax, errq):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        hd = 128
        C = (nq + 2 * nkv) * hd
        rng = np.random.default_rng(7)
        qkv_global = rng.standard_normal((L, C)).astype(np.float32)
        plan = mrsp.plan_shards(L, world).ranges
        b, e = plan[rank]
        mine = E.ulysses_plan(nq, nkv, world, rank)
        peers = [E.ulysses_plan(nq, nkv, world, p) for p in range(world)]
        Cme = (mine["q"][1] - mine["q"][0] + 2 * (mine["kv"][1] - mine["kv"][0])) * hd
        local = qkv_global[b:e]
        # ---- forward all-to-all (sequence shards -> head shards)
        qh = np.zeros((L, Cme), dtype=np.float32)
        reqs = []
        for p in range(world):
            Cp = (peers[p]["q"][1] - peers[p]["q"][0] + 2 * (peers[p]["kv"][1] - peers[p]["kv"][0])) * hd
            blk = np.zeros((e - b, Cp), dtype=np.float32)
            for src, dst, w in peers[p]["blocks"]:
                blk[:, dst:dst + w] = local[:, src:src + w]
            if p == rank:
                qh[b:e] = blk
            else:
                reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(blk)), p))
        for p in range(world):
            if p == rank:
                continue
            pb, pe = plan[p]
            buf = torch.empty((pe - pb, Cme))
            dist.recv(buf, p)
            qh[pb:pe] = buf.numpy()
        for r in reqs:
            r.wait()
        # head shard must equal the global rows restricted to my heads
        want = np.concatenate([qkv_global[:, s:s + w] for s, _, w in mine["blocks"]], axis=1)
        assert np.array_equal(qh, want), "forward all-to-all layout"
        # ---- attention on my heads (oracle math)
        nq_r = mine["q"][1] - mine["q"][0]
        nkv_r = mine["kv"][1] - mine["kv"][0]
        mask = T.mrsp_mask(L, Lp, Lmax)
        if nq_r:
            q = qh[:, : nq_r * hd].reshape(L, nq_r, hd).transpose(1, 0, 2).astype(np.float64)
            k = qh[:, nq_r * hd:(nq_r + nkv_r) * hd].reshape(L, nkv_r, hd).transpose(1, 0, 2).astype(np.float64)
            v = qh[:, (nq_r + nkv_r) * hd:].reshape(L, nkv_r, hd).transpose(1, 0, 2).astype(np.float64)
            if nkv_r == 1:
                k, v = np.repeat(k, nq_r, 0), np.repeat(v, nq_r, 0)
            oh = T.attention(q, k, v, mask, 0.1).transpose(1, 0, 2).reshape(L, nq_r * hd)
        else:
            oh = np.zeros((L, 0))
        # ---- backward all-to-all (head shards -> sequence shards)
        ol = np.zeros((e - b, nq * hd))
        reqs = []
        for p in range(world):
            pb, pe = plan[p]
            if p == rank:
                ol[:, mine["q"][0] * hd: mine["q"][1] * hd] = oh[b:e]
            elif nq_r:
                reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(oh[pb:pe])), p))
        for p in range(world):
            if p == rank:
                continue
            nq_p = peers[p]["q"][1] - peers[p]["q"][0]
            if not nq_p:
                continue
            buf = torch.empty((e - b, nq_p * hd), dtype=torch.float64)
            dist.recv(buf, p)
            ol[:, peers[p]["q"][0] * hd: peers[p]["q"][1] * hd] = buf.numpy()
        for r in reqs:
            r.wait()
        # ---- single-rank reference
        q = qkv_global[:, : nq * hd].reshape(L, nq, hd).transpose(1, 0, 2).astype(np.float64)
        k = qkv_global[:, nq * hd:(nq + nkv) * hd].reshape(L, nkv, hd).transpose(1, 0, 2).astype(np.float64)
        v = qkv_global[:, (nq + nkv) * hd:].reshape(L, nkv, hd).transpose(1, 0, 2).astype(np.float64)
        full = T.attention(q, k, v, mask, 0.1).transpose(1, 0, 2).reshape(L, nq * hd)
        assert np.allclose(ol, full[b:e], rtol=0, atol=1e-12), "backward all-to-all layout"
        # ---- Stage 1: frame plan + padded all-gather + compaction
        F, Tt, d = 11, 3, 5
        emb = rng.standard_normal((F * Tt, d))
        fplan = mrsp.plan_shards(F, world).ranges
        chunk = -(-F // world)
        fb, fe = fplan[rank]
        send = np.zeros((chunk * Tt, d))
        send[: (fe - fb) * Tt] = emb[fb * Tt: fe * Tt]
        out = [torch.empty((chunk * Tt, d), dtype=torch.float64) for _ in range(world)]
        dist.all_gather(out, torch.from_numpy(send))
        got = np.concatenate([out[w].numpy()[: (fplan[w][1] - fplan[w][0]) * Tt] for w in range(world)])
        assert np.array_equal(got, emb), "stage-1 gather compaction"
        dist.barrier()
        dist.destroy_process_group()
    except Exception as ex:  # surface the failure to the parent
        import traceback
        errq.put(f"rank {rank}: {ex}\n{traceback.format_exc()}")
        raise


@pytest.mark.parametrize("world,nq,nkv", [(2, 28, 4), (4, 28, 4), (4, 4, 2), (8, 28, 4)])
def test_ulysses_exchange_gloo(world, nq, nkv):
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    L, Lp, Lmax = 301, 201, 25  # uneven token shards, odd prefix, 4 rows
    mp.start_processes(_worker, args=(world, _free_port(), nq, nkv, L, Lp, Lmax, errq),
                       nprocs=world, join=True, start_method="spawn")
    assert errq.empty(), errq.get()


def test_head_split_covers_all_heads():
    for nq, nkv in ((28, 4), (4, 2), (16, 16)):
        for k in (1, 2, 4, 8, 16):
            if (k <= nkv and (nkv % k or nq % k)) or (k > nkv and k % nkv):
                with pytest.raises(Exception):
                    E.ulysses_plan(nq, nkv, k, 0)
                continue
            qs = []
            for r in range(k):
                p = E.ulysses_plan(nq, nkv, k, r)
                qs += list(range(*p["q"]))
                assert p["kv"][1] > p["kv"][0]
                for qh in range(*p["q"]):  # every local q head maps to a local kv head
                    assert p["kv"][0] <= qh // (nq // nkv) < p["kv"][1]
            assert sorted(qs) == list(range(nq)), (nq, nkv, k)
