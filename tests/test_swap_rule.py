"""The scatter's sibling swap pre-dedup (wavefront.cu, k_exact_scatter /
k_route) restated on the CPU and checked against the oracle's
layers: over windows of 32 (and 64 = adjacent tile pairs) consecutive
parents, a child that a lower-index parent of the window also offers is
dropped by the higher one. The rule must never drop a key's minimum-rank
emission (rank = idx*64 + v, dp.cpp:66), so the deduplicated next layer —
each key with its min-rank parent and vertex — is unchanged. Oracle only
(test infrastructure), no GPU."""
import pytest

from checkers import Oracle
from paper_1709_09990_b200 import generators as G


def offered(o, rows, k, layer):
    n = len(rows)
    out = []
    for s in layer:
        m = 0
        for v in range(n):
            if not (s >> v) & 1 and bin(o.q_set(rows, s, v)).count("1") <= k:
                m |= 1 << v
        out.append(m)
    return out


def swap_drops(sets, masks, window):
    """The kernel's rule: parent j drops w when some i < j of its window has
    S_i ^ S_j = {v, w} (v in S_j, w in S_i) and offers v."""
    kept = list(masks)
    for j, (sj, mj) in enumerate(zip(sets, masks)):
        base = (j // window) * window
        drop = 0
        for i in range(base, j):
            x = sets[i] ^ sj
            if bin(x).count("1") == 2 and masks[i] & x & sj:
                drop |= x & sets[i]
        kept[j] = mj & ~drop
    return kept


def min_rank_children(sets, masks):
    best = {}
    for idx, (s, m) in enumerate(zip(sets, masks)):
        x = m
        while x:
            v = (x & -x).bit_length() - 1
            x &= x - 1
            key = s | (1 << v)
            rank = idx * 64 + v
            if key not in best or rank < best[key]:
                best[key] = rank
    return best


@pytest.mark.parametrize("seed,n,p,k", [(1, 30, 0.25, 10), (3, 28, 0.3, 11), (5, 26, 0.35, 12)])
def test_swap_rule_keeps_min_rank_children(seed, n, p, k):
    o = Oracle()
    rows = G.random_graph(seed, n, p)
    run = o.decide(rows, k)
    checked = 0
    for layer in run.layers:
        sets = [s for s, _ in layer][:3000]
        if len(sets) < 64:
            continue
        masks = offered(o, rows, k, sets)
        want = min_rank_children(sets, masks)
        for window in (32, 64):
            kept = swap_drops(sets, masks, window)
            assert min_rank_children(sets, kept) == want
            assert sum(bin(m).count("1") for m in kept) <= sum(bin(m).count("1") for m in masks)
        checked += 1
        if checked == 3:
            break
    assert checked > 0
