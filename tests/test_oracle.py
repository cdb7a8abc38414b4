"""Pins the CPU oracle (oracle/etw_oracle.c) before anything trusts it:
against the reference's own known-answer tests (proj/tests/test_bloom.cpp,
test_dp.cpp, test_mmw.cpp), the golden vectors produced by the reference
(tests/golden/goldens.json), and — where oracle/_ref exists — the reference
library itself on randomized inputs. CPU only."""
import hashlib
import json
import math

import pytest

from paper_1709_09990_b200 import generators as G


def test_murmur3_published_vectors(oracle, goldens):
    # proj/tests/test_bloom.cpp:20-34
    assert oracle.murmur3(b"", 0) == 0
    assert oracle.murmur3(b"", 1) == 0x514E28B7
    assert oracle.murmur3(b"", 0xFFFFFFFF) == 0x81F16F39
    assert oracle.murmur3(b"\0\0\0\0", 0) == 0x2362F9DE
    assert oracle.murmur3(b"a", 0x9747B28C) == 0x7FA09EA6
    assert oracle.murmur3(b"Hello, world!", 0x9747B28C) == 0x24884CBA
    for data_hex, seed, value in goldens["murmur3"]:
        assert oracle.murmur3(bytes.fromhex(data_hex), seed) == value


def test_hash_pairs_are_frozen(oracle, goldens):
    # proj/tests/test_bloom.cpp:36-44
    assert oracle.hash_pair(0) == (0x2E1D9BD8, 0x94AF0861)
    assert oracle.hash_pair(1) == (0x24E81313, 0x6CA67478)
    assert oracle.hash_pair(0x0123456789ABCDEF) == (0xD91B202A, 0x143C713C)
    assert oracle.hash_pair(0xFFFFFFFFFFFFFFFF) == (0x7584C82B, 0x1C6FD6CF)
    for key, h1, h2 in goldens["hash_pair"]:
        assert oracle.hash_pair(key) == (h1, h2)


def test_bloom_sizing_and_fp_formula(oracle, goldens):
    # test_bloom.cpp:58-64, 96-104
    L = oracle.lib
    assert L.oracle_bloom_bits(1000, 24) >= 24000 and L.oracle_bloom_bits(1000, 24) % 64 == 0
    assert L.oracle_bloom_bits(0, 24) == 64
    m = L.oracle_bloom_bits(1_000_000, 24)
    assert math.isclose(L.oracle_bloom_expected_fp(m, 17, 1_000_000), 9.838577e-06, rel_tol=0.01)
    assert math.isclose(L.oracle_bloom_expected_fp(m, 17, 2_000_000), 8.898144e-03, rel_tol=0.01)
    assert math.isclose(L.oracle_bloom_expected_fp(m, 17, 1_000_000), goldens["bloom_fp"]["1e6@1e6"],
                        rel_tol=1e-12)


def test_bloom_sequence_matches_reference(oracle, goldens):
    stream = [(i * 0x9E3779B97F4A7C15) & (2**64 - 1) for i in range(3000)]
    stream += stream[::7]
    m, novel = oracle.bloom_insert_seq(1000, stream)
    g = goldens["bloom_seq"]
    assert m == g["m"]
    assert sum(novel) == g["novel_count"]
    assert hashlib.sha256(bytes(novel)).hexdigest() == g["novel_digest"]
    # insert twice reports novel exactly once (test_bloom.cpp:66-73)
    _, nv = oracle.bloom_insert_seq(100, [42, 42, 43])
    assert nv == [True, False, True]


def test_q_set_walks_through_eliminated(oracle):
    p3 = G.path_graph(3)  # test_graph.cpp:158-163
    assert oracle.q_set(p3, 0b010, 0) == 0b100
    assert oracle.q_set(p3, 0b010, 2) == 0b001
    g = G.random_graph(7, 8, 0.5)
    for v in range(8):
        assert oracle.q_set(g, 0, v) == g[v]


def _triangle_states():
    return [(1 << v, (0xFFFFFFFF << 8 | v) & 0xFFFFFFFF) for v in range(3)]


def test_expand_layer_known_answers(oracle):
    k3 = G.complete_graph(3)
    # root of K3 at k=2 (test_dp.cpp:66-83)
    for mode in ("bloom", "exact"):
        r = oracle.expand_layer(k3, 2, [(0, 0xFFFFFFFF)], dedup=mode)
        assert sorted(s for s, _ in r.layers[0]) == [1, 2, 4]
        assert r.rounds[0].tuple()[2:5] == (1, 3, 0)
    # converging paths (test_dp.cpp:94-106)
    r = oracle.expand_layer(k3, 2, _triangle_states(), dedup="exact")
    assert sorted(s for s, _ in r.layers[0]) == [3, 5, 6]
    assert (r.rounds[0].expanded, r.rounds[0].emitted, r.rounds[0].duplicates) == (3, 3, 3)
    # first emission wins (test_dp.cpp:108-120)
    r = oracle.expand_layer(k3, 2, _triangle_states()[:2], dedup="exact")
    assert [s for s, _ in r.layers[0]] == [3, 5, 6]
    assert r.layers[0][0][1] == ((0xFFFFFF00 | 0) << 8 | 1) & 0xFFFFFFFF
    # capacity keeps the oldest (test_dp.cpp:132-143)
    star = G.biclique(1, 3)
    for mode in ("bloom", "exact"):
        r = oracle.expand_layer(star, 1, [(0, 0xFFFFFFFF)], dedup=mode, cap=2)
        assert r.overflowed and sorted(s for s, _ in r.layers[0]) == [2, 4]
    # forbidden (test_dp.cpp:122-130)
    r = oracle.expand_layer(G.path_graph(4), 1, [(0, 0xFFFFFFFF)], forbidden=0b1010, dedup="exact")
    assert [s for s, _ in r.layers[0]] == [1]


def _smallest_k(oracle, rows, **kw):
    for k in range(len(rows)):
        r = oracle.decide(rows, k, keep_layers=False, **kw)
        assert r.outcome != "indeterminate"
        if r.outcome == "feasible":
            return k
    return max(0, len(rows) - 1)


def test_decide_known_treewidths(oracle):
    # test_dp.cpp:162-168
    assert _smallest_k(oracle, G.path_graph(5)) == 1
    assert _smallest_k(oracle, G.cycle_graph(6), dedup="bloom") == 2
    assert _smallest_k(oracle, G.grid_graph(3, 3)) == 3
    assert _smallest_k(oracle, G.petersen_graph(), dedup="bloom") == 4
    assert _smallest_k(oracle, G.biclique(3, 3)) == 3
    r = oracle.decide(G.path_graph(4), 1, forbidden=0b1100, rounds=2)  # test_dp.cpp:283-290
    assert r.outcome == "feasible" and r.witness_set == 3 and len(r.rounds) == 2


def test_mmw_knowns(oracle):
    # test_mmw.cpp:97-106
    assert oracle.mmw_lower_bound(G.complete_graph(4)) == 3
    assert oracle.mmw_lower_bound(G.complete_graph(6)) == 5
    assert oracle.mmw_lower_bound(G.cycle_graph(6)) == 2
    assert oracle.mmw_lower_bound(G.path_graph(5)) == 1
    # contract step on K4 (test_mmw.cpp:73-85): v=0 u=1 common=2 min_after=2
    bound, steps = oracle.mmw_trace(G.complete_graph(4))
    assert steps[0][:4] == (0, 1, 2, 2)


def test_instance_goldens_through_oracle(oracle, goldens):
    """myciel4: the oracle's deepening loop (clique forbidden, no improvement
    edges) lands on the reference's treewidth."""
    g = goldens["instances"]["myciel4"]
    clique = g["max_clique"]
    k0 = max(bin(clique).count("1") - 1, g["mmw_root"])
    k, _ = oracle.deepen(G.myciel(4), k0, forbidden=clique)
    assert k == g["tw"] == 10


def test_oracle_matches_reference_decide(oracle, ref):
    """Layer-by-layer identity (sets, order, histories, counters) with the
    reference's decide on random graphs, every mode (dp.cpp:73-194)."""
    for seed in range(60):
        n = 4 + seed % 9
        rows = G.random_graph(seed * 131 + 5, n, 0.2 + 0.1 * (seed % 6))
        for k in range(0, n, 2):
            for dedup in ("exact", "bloom"):
                for mmw in (False, True):
                    cap = 3 if seed % 5 == 0 else 10_000_000
                    a = ref.decide(rows, k, dedup=dedup, mmw=mmw, cap=cap)
                    b = oracle.decide(rows, k, dedup=dedup, mmw=mmw, cap=cap)
                    assert (a.outcome, a.witness_set, a.witness_hist, a.overflowed) == \
                        (b.outcome, b.witness_set, b.witness_hist, b.overflowed)
                    assert [x.tuple() for x in a.rounds] == [x.tuple() for x in b.rounds]
                    assert a.layers == b.layers


def test_oracle_mmw_trace_matches_reference(oracle, ref):
    import random
    rng = random.Random(33)
    for it in range(200):
        n = 2 + rng.randrange(12)
        rows = G.random_graph(rng.randrange(1 << 30), n, 0.15 + 0.1 * (it % 8))
        s = rng.randrange(1 << n) if it % 2 else 0
        cap = rng.randrange(4) if it % 3 == 0 else 2**31 - 1
        assert oracle.mmw_trace(rows, s, cap) == ref.mmw_trace(rows, s, cap)


def test_oracle_myciel4_layers_match_golden_digest(oracle, goldens, ref):
    """The reference's solve layer log for myciel4 (exact) reproduced by the
    oracle decide on the reference's improved graphs."""
    g = goldens["instances"]["myciel4"]
    rows = G.myciel(4)
    clique = g["max_clique"]
    stats = json.loads(g["exact_stats"])
    layers = []
    for att in stats["components"][0]["attempts"]:
        gk = ref.improve_graph(rows, att["k"])
        r = oracle.decide(gk, att["k"], forbidden=clique)
        assert [x.emitted for x in r.rounds] == [x["emitted"] for x in att["layers"]]
        assert [x.duplicates for x in r.rounds] == [x["duplicates"] for x in att["layers"]]
        layers += r.layers
    from golden.make_goldens import layer_digest
    assert layer_digest(layers) == g["exact_layer_digest"]
