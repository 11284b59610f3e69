"""GPU: the production head geometry at SP = 8 (28 query / 4 kv heads, hd 128:
every kv head replicated to a rank pair) on a narrow model, end to
end. The pair splits the kv head's work by query rows — each rank all 7 query
heads over half of the 256-row query blocks, dealt by causal cost
(mrsp_attn_row_part; the default of the fused transports) — or, with
MRSP_ULYSSES_SPLIT=heads, by query heads 4 + 3 (the NCCL transport's plan).
8 virtual ranks in one process (both splits) and 8 processes sharing one B200
through CUDA-IPC peer memory (the transport the N = 8 bench uses) are
bit-identical to SP = 1, and close to the oracle."""
import numpy as np
import pytest

from oracle import transformer as T
from paper_2507_07966_b200 import engine as E

import test_p2p_gpu as P

pytestmark = pytest.mark.gpu

# c1's tiny vision tower with a 28 / 4-head LLM (dim 256, 2 layers, V 32)
CFG = E._cfg(image_size=64, patch=8, v_dim=256, v_heads=4, v_head_dim=64, v_mlp=1024, v_layers=2,
             dim=256, n_q_heads=28, n_kv_heads=4, mlp=1024, layers=2, vocab=32)
W = E.Workload("sp8geo", CFG, 8, 8, 4, 3, 6, 12, "28/4 heads at SP=8")


def _inputs():
    pix = E.gen_video(1, W.frames, 3 * CFG.image_size ** 2)
    grp = E.make_group(W, seed=3)
    return pix, grp


def _run_local(sp, pix, grp):
    eng = E.Engine(CFG, sp=sp, vision_seed=2, policy_seed=3, ref_seed=4)
    eng.encode("v", pix)
    out = eng.step("v", pix, grp, with_kl=True)
    eng.close()
    return out


def test_plan_is_the_production_split():
    plans = [E.ulysses_plan(28, 4, 8, r) for r in range(8)]
    assert [p["q"][1] - p["q"][0] for p in plans] == [4, 3] * 4
    assert [p["kv"] for p in plans] == [(g, g + 1) for g in range(4) for _ in range(2)]


@pytest.mark.parametrize("split", ["rows", "heads"])
def test_sp8_virtual_ranks_bit_exact_and_oracle(gpu, split, monkeypatch):
    monkeypatch.setenv("MRSP_ULYSSES_SPLIT", split)
    pix, grp = _inputs()
    base = _run_local(1, pix, grp)
    got = _run_local(8, pix, grp)
    for a, b in zip(base, got):
        assert np.array_equal(a, b)
    c = T.Cfg.from_any(CFG)
    emb = T.vision_forward(c, T.vision_weights(c, 2), pix)
    want, _ = T.llm_logprobs(c, T.llm_weights(c, 3, "policy."), emb, grp.question, grp.resp,
                             grp.lengths)
    d = np.abs(base[0] - want)
    assert d.max() <= 5e-2 and d.mean() <= 5e-3, (d.max(), d.mean())


def _worker(rank, world, port, q):
    import os
    try:
        import torch
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        pix, grp = _inputs()
        eng = E.Engine(CFG, sp=world, rank=rank, n_procs=world, vision_seed=2, policy_seed=3,
                       ref_seed=4)
        L = W.frames * CFG.tokens_per_frame + len(grp.question) + grp.resp.shape[0] * grp.Lmax
        blobs = [None] * world
        dist.all_gather_object(blobs, eng.p2p_export(W.frames, L, grp.scored))
        eng.p2p_import(blobs)
        eng.encode("v", pix)
        out = eng.step("v", pix, grp, with_kl=True)
        out = tuple(out) + tuple(eng.generate("v", grp.question, 4, 12, temperature=1.0, seed=5))
        dist.barrier()
        eng.close()
        dist.destroy_process_group()
        q.put((rank, out, None))
    except Exception as ex:
        q.put((rank, None, repr(ex)))


def test_sp8_processes_p2p_bit_exact(gpu):
    """... and rollout generation in the 8-process engine (prompt K/V gathered
    from the peers' head shards over CUDA-IPC) is bit-identical to SP = 1."""
    import multiprocessing as mp
    pix, grp = _inputs()
    eng = E.Engine(CFG, sp=1, vision_seed=2, policy_seed=3, ref_seed=4)
    eng.encode("v", pix)
    base = tuple(eng.step("v", pix, grp, with_kl=True)) + tuple(
        eng.generate("v", grp.question, 4, 12, temperature=1.0, seed=5))
    eng.close()
    ctx = mp.get_context("spawn")
    qu = ctx.Queue()
    port = P._free_port()
    procs = [ctx.Process(target=_worker, args=(r, 8, port, qu)) for r in range(8)]
    for p in procs:
        p.start()
    res = sorted([qu.get(timeout=900) for _ in range(8)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
    for rank, out, err in res:
        assert err is None, f"rank {rank}: {err}"
        for a, b in zip(base, out):
            assert np.array_equal(a, b), f"rank {rank} differs from SP=1"
