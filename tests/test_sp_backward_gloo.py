"""CPU, multi-process (gloo): the sequence-parallel routing of the attention
BACKWARD (csrc/engine_bwd.cu + the route kernels of csrc/backward.cu) restated
with the library's own plans, one process per SP rank.

Each rank holds a sequence shard (plan_shards) and, by the engine's head split
(mrsp_head_split: whole heads up to the kv-head count, the query-row split of
256-row blocks above it, mrsp_attn_row_part), a head shard:
  1. sequence -> heads: dO columns of each rank's query heads (the engine sends
     the row dots D = rowsum(dO o O) along the same routes), only for the rows
     of the owner's row blocks;
  2. the attention backward on the head shard (float64 numpy): dQ for the own
     rows, dK / dV partial over them;
  3. heads -> sequence: dq rows to the token owners; dk / dv rows directly, or,
     for a kv head shared by m ranks, into slot (rank % m) of the owner, which
     sums its m slots in slot order.
The assembled dq / dk / dv must equal the single-rank backward of the MR-SP
attention (causal prefix + rollout rows, GQA) to float64 rounding.
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

HD = 128


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def attn_bwd(q, k, v, dO, mask, rows=None):
    """float64 backward of softmax(mask(q k^T / sqrt(hd))) v for GQA, q [L, nq, hd],
    k / v [L, nkv, hd]; only query rows in `rows` (bool [L]) contribute."""
    L, nq, _ = q.shape
    nkv = k.shape[1]
    rep = nq // nkv
    scale = 1 / np.sqrt(HD)
    dq, dk, dv = np.zeros_like(q), np.zeros_like(k), np.zeros_like(v)
    use = np.ones(L, bool) if rows is None else rows
    for h in range(nq):
        g = h // rep
        s = (q[:, h] @ k[:, g].T) * scale
        s = np.where(mask, s, -np.inf)
        p = np.exp(s - s.max(1, keepdims=True))
        p /= p.sum(1, keepdims=True)
        o = p @ v[:, g]
        D = (dO[:, h] * o).sum(1, keepdims=True)
        dp = dO[:, h] @ v[:, g].T
        ds = p * (dp - D)
        ds[~use] = 0.0
        pu = np.where(use[:, None], p, 0.0)
        dq[:, h] = np.where(use[:, None], ds @ k[:, g] * scale, 0.0)
        dk[:, g] += ds.T @ q[:, h] * scale
        dv[:, g] += pu.T @ dO[:, h]
    return dq, dk, dv


def _inputs(L, nq, nkv):
    rng = np.random.default_rng(11)
    q = rng.standard_normal((L, nq, HD))
    k = rng.standard_normal((L, nkv, HD))
    v = rng.standard_normal((L, nkv, HD))
    dO = rng.standard_normal((L, nq, HD))
    return q, k, v, dO


def _worker(rank, world, port, nq, nkv, L, Lp, Lmax, row_split, errq):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        q, k, v, dO = _inputs(L, nq, nkv)
        mask = T.mrsp_mask(L, Lp, Lmax)
        plan = mrsp.plan_shards(L, world).ranges
        hs = [E.head_split(nq, nkv, world, p, row_split) for p in range(world)]
        n_blocks = (L + 255) // 256
        m_kv = world // nkv if world > nkv else 1

        def owns_row(p, row):
            h = hs[p]
            return h["row_parts"] == 1 or \
                E.attn_row_part(row // 256, n_blocks, h["row_parts"]) == h["row_part"]

        b, e = plan[rank]
        me = hs[rank]
        q0, q1 = me["q"]
        k0, k1 = me["kv"]
        # 1. sequence -> heads: this shard's dO (its rows, every rank's heads)
        doh = np.zeros((L, q1 - q0, HD))
        reqs = []
        for p in range(world):
            pq0, pq1 = hs[p]["q"]
            rows = np.array([r for r in range(b, e) if owns_row(p, r)], dtype=np.int64)
            blk = dO[rows][:, pq0:pq1] if len(rows) else np.zeros((0, pq1 - pq0, HD))
            if p == rank:
                doh[rows] = blk
            else:
                reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(blk)), p))
        for p in range(world):
            if p == rank:
                continue
            pb, pe = plan[p]
            rows = np.array([r for r in range(pb, pe) if owns_row(rank, r)], dtype=np.int64)
            buf = torch.zeros((len(rows), q1 - q0, HD), dtype=torch.float64)
            dist.recv(buf, p)
            doh[rows] = buf.numpy()
        for r_ in reqs:
            r_.wait()
        # 2. attention backward on the head shard (own rows only)
        own = np.array([owns_row(rank, r) for r in range(L)])
        dq_h, dk_h, dv_h = attn_bwd(q[:, q0:q1], k[:, k0:k1], v[:, k0:k1], doh, mask, own)
        # 3. heads -> sequence: dq rows; dk / dv rows (direct or slot partials)
        dq = np.zeros((e - b, nq, HD))
        slots = np.zeros((m_kv, e - b, nkv, 2, HD))
        reqs = []
        for p in range(world):
            pb, pe = plan[p]
            payload = np.concatenate([dq_h[pb:pe].reshape(pe - pb, -1),
                                      dk_h[pb:pe].reshape(pe - pb, -1),
                                      dv_h[pb:pe].reshape(pe - pb, -1)], 1)
            if p == rank:
                mine = payload
            else:
                reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(payload)), p))
        for p in range(world):
            pq0, pq1 = hs[p]["q"]
            pk0, pk1 = hs[p]["kv"]
            if p == rank:
                pay = mine
            else:
                buf = torch.zeros((e - b, (pq1 - pq0 + 2 * (pk1 - pk0)) * HD), dtype=torch.float64)
                dist.recv(buf, p)
                pay = buf.numpy()
            nqp, nkp = pq1 - pq0, pk1 - pk0
            dq_p = pay[:, :nqp * HD].reshape(e - b, nqp, HD)
            dk_p = pay[:, nqp * HD:(nqp + nkp) * HD].reshape(e - b, nkp, HD)
            dv_p = pay[:, (nqp + nkp) * HD:].reshape(e - b, nkp, HD)
            for i, row in enumerate(range(b, e)):
                if owns_row(p, row):
                    dq[i, pq0:pq1] = dq_p[i]
            slot = p % m_kv if m_kv > 1 else 0
            slots[slot, :, pk0:pk1, 0] += dk_p  # each (slot, kv head) written once
            slots[slot, :, pk0:pk1, 1] += dv_p
        for r_ in reqs:
            r_.wait()
        dkv = slots[0].copy()
        for j in range(1, m_kv):
            dkv += slots[j]
        want_q, want_k, want_v = attn_bwd(q, k, v, dO, mask)
        np.testing.assert_allclose(dq, want_q[b:e], rtol=0, atol=1e-10)
        np.testing.assert_allclose(dkv[:, :, 0], want_k[b:e], rtol=0, atol=1e-10)
        np.testing.assert_allclose(dkv[:, :, 1], want_v[b:e], rtol=0, atol=1e-10)
        dist.barrier()
        dist.destroy_process_group()
    except Exception as ex:  # surfaced by the parent
        errq.put(f"rank {rank}: {ex!r}")


@pytest.mark.parametrize("world,nq,nkv,row_split", [(2, 4, 2, True), (4, 4, 2, True),
                                                     (2, 7, 1, True), (2, 7, 1, False),
                                                     (8, 28, 4, True)])
def test_backward_routing_matches_single_rank(world, nq, nkv, row_split):
    """world 2 with 2 kv heads: whole heads per rank; world > kv heads: the
    query-row split (world 8 with 28 / 4 heads is c4's SP 8 of Qwen2.5-7B), or
    with row_split False the 4+3-style split of a replicated kv head's query
    heads — either way each kv head's dK / dV arrives as partials in slots."""
    Lp, Lmax, G = 300, 140, 3
    L = Lp + G * Lmax
    errq = mp.get_context("spawn").SimpleQueue()
    mp.start_processes(_worker, args=(world, _free_port(), nq, nkv, L, Lp, Lmax, row_split, errq),
                       nprocs=world, join=True, start_method="spawn")
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, errs
