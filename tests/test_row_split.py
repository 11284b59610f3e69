"""CPU: the query-row split the fused SP transports use when SP > n_kv
(mrsp_attn_row_part, csrc/common.h) — every 256-row query block has exactly one
owner among the m ranks sharing a kv head, and the owners' attention work
(visible 128-key tiles under the MR-SP mask, the kernel's own skip rule) is
balanced: at the c4 geometry the ranks of a pair differ by < 0.5% (the 4+3
query-head split it replaces: 4/3.5 = 14% above the mean). The reference's
balance contract is plan_shards' "at most one item of imbalance"
(/root/reference/proj/src/engine.cpp:15-29, idle fraction :271-277)."""
import numpy as np
import pytest

from paper_2507_07966_b200 import _lib


def part(b, n, m):
    return _lib.lib().mrsp_attn_row_part(b, n, m)


def block_cost(L, Lp, Lmax):
    """Visible KV tiles per 256-row block (two 128-row query tiles), counting a
    tile for each query tile that sees any key in it."""
    n_blocks = (L + 255) // 256
    cost = np.zeros(n_blocks)
    for b in range(n_blocks):
        for t in range(2):
            q0 = b * 256 + t * 128
            if q0 >= L:
                continue
            q1 = min(q0 + 127, L - 1)
            if q1 < Lp:
                cost[b] += q1 // 128 + 1
            else:  # rows: the prefix + (parts of) their own segments
                rows = {(q - Lp) // Lmax for q in range(max(q0, Lp), q1 + 1)}
                tiles = set(range((min(q1, Lp - 1)) // 128 + 1)) if q0 < Lp else set(range((Lp - 1) // 128 + 1))
                for r in rows:
                    lo = Lp + r * Lmax
                    tiles |= set(range(lo // 128, min(q1, lo + Lmax - 1) // 128 + 1))
                cost[b] += len(tiles)
    return cost


@pytest.mark.parametrize("n_blocks", [1, 2, 3, 7, 8, 9, 544])
@pytest.mark.parametrize("m", [1, 2, 3, 4])
def test_every_block_has_one_owner(n_blocks, m):
    owners = [part(b, n_blocks, m) for b in range(n_blocks)]
    assert all(0 <= o < m for o in owners)
    counts = np.bincount(owners, minlength=m)
    assert counts.max() - counts.min() <= 1


def test_bad_arguments():
    assert part(0, 0, 2) == -1 and part(5, 5, 2) == -1 and part(0, 4, 0) == -1


def test_c4_pair_balance():
    Lp, G, Lmax = 131109, 8, 1011
    L = Lp + G * Lmax
    cost = block_cost(L, Lp, Lmax)
    n = len(cost)
    for m in (2, 4):
        shares = np.zeros(m)
        for b in range(n):
            shares[part(b, n, m)] += cost[b]
        assert shares.max() / shares.mean() - 1 < 5e-3, (m, shares)
    # the head split it replaces: 4 of 7 query heads on one rank of the pair
    assert 4 / 3.5 - 1 > 0.14
