"""Test infrastructure: a plain-Python restatement of the owner-sharded round
protocol of paper_1709_09990_b200/csrc/shard.cu, run over torch.distributed
(gloo) on CPU processes so the N>1 path's host-side logic — ownership,
all-to-all routing, owner dedup with min-rank histories, the per-round count
allgather, shard-major truncation, termination — is exercised at world size 2
without a GPU. Candidate tests use the CPU oracle's q_set (graph.hpp:61-78);
nothing here is on the product path."""
MASK64 = (1 << 64) - 1


def fmix64(k: int) -> int:
    k &= MASK64
    k ^= k >> 33
    k = (k * 0xFF51AFD7ED558CCD) & MASK64
    k ^= k >> 33
    k = (k * 0xC4CEB9FE1A85EC53) & MASK64
    k ^= k >> 33
    return k


def owner_of(key: int, shards: int, words: int = 1) -> int:
    """shard.cu owner_of: mulhi(mix(S), G)."""
    h = fmix64((key & MASK64) ^ 0xD6E8FEB86659FD93)
    if words == 2:
        h = fmix64(h ^ (key >> 64))
    return (h * shards) >> 64


def _bits(x: int):
    while x:
        low = x & -x
        yield low.bit_length() - 1
        x ^= low


def sharded_decide(rows, k, q_set, dist, forbidden=0, cap=10_000_000, rounds=-1):
    """One shard's view of a decide; returns (per-round counters, this shard's
    final layer, outcome). Counters are (round, expanded, emitted, duplicates,
    overflowed), global across shards."""
    me, shards = dist.get_rank(), dist.get_world_size()
    n = len(rows)
    free = n - bin(forbidden).count("1")
    if rounds < 0:
        rounds = max(0, n - k - 1)
    layer = [(0, 0xFFFFFFFF)] if me == 0 else []  # the root starts on shard 0
    stats, overflow = [], False
    for r in range(rounds):
        outbox = [[] for _ in range(shards)]
        offered = 0
        for idx, (s, hist) in enumerate(layer):
            eligible = ((1 << n) - 1) & ~s & ~forbidden
            for v in _bits(eligible):
                if bin(q_set(rows, s, v)).count("1") <= k:  # dp.cpp:56
                    key = s | (1 << v)
                    rank = (me << 40) | (idx * 64 + v)
                    outbox[owner_of(key, shards)].append((key, rank, ((hist << 8) | v) & 0xFFFFFFFF))
                    offered += 1
        boxes = [None] * shards
        dist.all_gather_object(boxes, outbox)  # the all-to-all exchange
        best = {}
        for src in range(shards):
            for key, rank, hist in boxes[src][me]:
                if key not in best or rank < best[key][0]:
                    best[key] = (rank, hist)  # min-rank emission keeps its history
        mine = sorted((rank, key, hist) for key, (rank, hist) in best.items())
        counts = [None] * shards
        dist.all_gather_object(counts, (len(layer), offered, len(mine)))
        expanded = sum(c[0] for c in counts)
        offered_all = sum(c[1] for c in counts)
        unique = sum(c[2] for c in counts)
        cap_r = min(cap, max(1, expanded * free))  # dp.cpp:84-86
        emitted = min(unique, cap_r)
        before = sum(c[2] for c in counts[:me])
        keep = min(len(mine), max(0, cap_r - before))  # shard-major capacity wall
        layer = [(key, hist) for _, key, hist in mine[:keep]]
        overflow = overflow or unique > cap_r
        stats.append((r, expanded, emitted, offered_all - unique, unique > cap_r))
        if emitted == 0:
            return stats, layer, "indeterminate" if overflow else "infeasible"
    return stats, layer, "feasible"
