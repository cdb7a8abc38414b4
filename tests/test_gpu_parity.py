"""Device parity: the sm_100a wavefront (through the C ABI) against the CPU
oracle, the reference library (oracle/_ref) and the reference's golden
vectors. Exact mode must be bit-identical — every layer's states, their order,
their histories and every counter; Bloom mode must reach the same verdicts
and, absent false positives, the same state sets and counters."""
import json
import random

import pytest

from conftest import instance_text
from paper_1709_09990_b200 import generators as G

pytestmark = pytest.mark.gpu


def _norm(run):
    return (run.outcome, run.witness_set, run.witness_hist, run.overflowed,
            [x.tuple() for x in run.rounds], run.layers)


def _triangle_states():
    return [(1 << v, (0xFFFFFF00 | v)) for v in range(3)]


def test_expand_layer_known_answers(E, gpu):
    k3 = G.complete_graph(3)
    for mode in ("bloom", "exact"):  # test_dp.cpp:66-83
        r = E.expand_layer(k3, 2, [(0, 0xFFFFFFFF)], dedup=mode)
        assert sorted(s for s, _ in r.layers[0]) == [1, 2, 4]
        assert (r.rounds[0].expanded, r.rounds[0].emitted, r.rounds[0].duplicates) == (1, 3, 0)
        for s, h in r.layers[0]:
            assert h == (0xFFFFFF00 | (s.bit_length() - 1))
    r = E.expand_layer(G.biclique(1, 3), 1, [(0, 0xFFFFFFFF)], dedup="exact")  # :85-92
    assert sorted(s for s, _ in r.layers[0]) == [2, 4, 8]
    r = E.expand_layer(k3, 2, _triangle_states(), dedup="exact")  # :94-106
    assert sorted(s for s, _ in r.layers[0]) == [3, 5, 6]
    assert (r.rounds[0].expanded, r.rounds[0].emitted, r.rounds[0].duplicates) == (3, 3, 3)
    r = E.expand_layer(k3, 2, _triangle_states()[:2], dedup="exact")  # :108-120
    assert [s for s, _ in r.layers[0]] == [3, 5, 6]
    assert r.layers[0][0][1] == (((0xFFFFFF00 | 0) << 8) | 1) & 0xFFFFFFFF
    r = E.expand_layer(G.path_graph(4), 1, [(0, 0xFFFFFFFF)], forbidden=0b1010)  # :122-130
    assert [s for s, _ in r.layers[0]] == [1]
    for mode in ("bloom", "exact"):  # :132-143
        r = E.expand_layer(G.biclique(1, 3), 1, [(0, 0xFFFFFFFF)], dedup=mode, cap=2)
        assert r.overflowed and r.rounds[0].overflowed
        assert sorted(s for s, _ in r.layers[0]) == [2, 4]


def test_expand_layer_matches_oracle_on_mixed_inputs(E, oracle, gpu):
    rng = random.Random(3)
    for it in range(40):
        n = 6 + it % 40
        rows = G.random_graph(it + 100, n, 0.3)
        states = []
        for _ in range(1 + it * 3):
            s = 0
            for v in range(n):
                if rng.random() < 0.3:
                    s |= 1 << v
            states.append((s, rng.getrandbits(32)))
        for mode in ("exact",):
            a = E.expand_layer(rows, 4 + it % 6, states, dedup=mode)
            b = oracle.expand_layer(rows, 4 + it % 6, states, dedup=mode)
            assert a.layers == b.layers
            assert [x.tuple()[2:] for x in a.rounds] == [x.tuple()[2:] for x in b.rounds]


def test_decide_matches_oracle_exact(E, oracle, gpu):
    """Identical layers (order + histories), counters and witness."""
    for seed in range(60):
        n = 4 + seed % 22
        rows = G.random_graph(seed * 131 + 5, n, 0.15 + 0.05 * (seed % 8))
        for k in sorted({max(0, n // 4), n // 3}):
            for mmw in (False, True) if n <= 14 else (False,):
                cap = 5 if seed % 7 == 0 else 10_000_000
                a = E.decide(rows, k, dedup="exact", mmw=mmw, cap=cap)
                b = oracle.decide(rows, k, dedup="exact", mmw=mmw, cap=cap)
                assert _norm(a) == _norm(b), (seed, k, mmw, cap)


def test_decide_forbidden_and_explicit_rounds(E, oracle, gpu):
    r = E.decide(G.path_graph(4), 1, forbidden=0b1100, rounds=2)  # test_dp.cpp:283-290
    assert r.outcome == "feasible" and r.witness_set == 3 and len(r.rounds) == 2
    for n in (1, 2, 4, 6):  # complete graphs need zero rounds (test_dp.cpp:145-152)
        r = E.decide(G.complete_graph(n), n - 1, forbidden=(1 << n) - 1)
        assert r.outcome == "feasible" and r.rounds == [] and r.witness_set == 0
    r = E.decide(G.complete_graph(4), 2)
    assert r.outcome == "infeasible" and not r.overflowed
    for seed in range(20):
        rows = G.random_graph(seed, 14, 0.35)
        f = random.Random(seed).getrandbits(14) & 0b10100101001010
        a = E.decide(rows, 5, forbidden=f, rounds=6)
        b = oracle.decide(rows, 5, forbidden=f, rounds=6)
        assert _norm(a) == _norm(b)


def test_decide_validates_configuration(E, gpu):
    with pytest.raises(ValueError):
        E.decide(G.path_graph(3), -1)
    with pytest.raises(ValueError):
        E.decide(G.path_graph(3), 1, cap=0)


def test_decide_bloom_agrees_with_oracle(E, oracle, gpu):
    """Bloom layers depend on insertion order (a key whose h2 is 0 mod m
    probes one bit 17 times, e.g. 0x220d at m=336960), exactly as in the
    reference at >1 thread (docs/stats-schema.md:16-18). What must hold:
    the verdict, exactly-once novelty (no duplicate states in a layer), and
    every Bloom layer is a subset of the exact layer of the same round, short
    by at most a few false positives."""
    for seed in range(30):
        n = 6 + seed % 18
        rows = G.random_graph(seed * 17 + 3, n, 0.2 + 0.04 * (seed % 6))
        for k in (n // 4, n // 3):
            a = E.decide(rows, k, dedup="bloom")
            b = oracle.decide(rows, k, dedup="exact")
            assert a.outcome == b.outcome
            assert len(a.rounds) == len(b.rounds)
            for la, lb, ra in zip(a.layers, b.layers, a.rounds):
                sa = {s for s, _ in la}
                assert len(sa) == len(la) == ra.emitted
                assert sa <= {s for s, _ in lb}
                assert len(sa) >= len(lb) - max(2, len(lb) // 100)
            # with the lock and warp pre-dedup disabled/forced the same holds
    _, nv = oracle.bloom_insert_seq(14040, [0x220D])
    assert oracle.hash_pair(0x220D)[1] % 336960 == 0 and nv == [True]


def test_wide_masks_match_oracle(E, oracle, gpu):
    """n > 64 takes the 128-bit path (Set<2>, 16-byte keys); no reference
    exists, the oracle restatement is the checker."""
    for i, n in enumerate((66, 72, 80, 96, 112, 128)):
        rows = G.random_graph(i + 7, n, 8.0 / n)
        for dedup in ("exact", "bloom"):
            a = E.decide(rows, 5, dedup=dedup, rounds=6)
            b = oracle.decide(rows, 5, dedup=dedup, rounds=6)
            if dedup == "exact":
                assert _norm(a) == _norm(b)
            else:
                assert a.outcome == b.outcome
                assert [sorted(s for s, _ in x) for x in a.layers] == \
                    [sorted(s for s, _ in x) for x in b.layers]
    rows = G.grid_with_chords(8, 9, 6, 7)
    for k, rounds in ((4, 6), (8, 2)):
        a = E.decide(rows, k, dedup="exact", rounds=rounds, mmw=True)
        b = oracle.decide(rows, k, dedup="exact", rounds=rounds, mmw=True)
        assert _norm(a) == _norm(b)


def test_instances_exact_stats_are_byte_identical(E, goldens, gpu):
    """etw_solve in exact mode with order reconstruction: the JSON report
    (every layer counter, reconstruction_expanded, the order) equals the
    reference's byte for byte (solver.cpp:198-297)."""
    for name, g in goldens["instances"].items():
        graph = E.Graph.parse(instance_text(name))
        res = E.solve(graph, E.Options(dedup="exact", emit_order=True))
        assert res.kind == "exact" and res.value == g["tw"]
        assert res.order == g["exact_order"]
        assert res.stats_json == g["exact_stats"], name
        w, ok = graph.check_order(res.order)
        assert ok and w == g["tw"]


def test_instances_layer_logs_match_reference(E, goldens, gpu):
    from golden.make_goldens import layer_digest
    for name, g in goldens["instances"].items():
        run = E.solve_layers(E.Graph.parse(instance_text(name)), E.Options(dedup="exact"))
        assert [len(x) for x in run.layers] == g["exact_layer_sizes"]
        assert [list(t) for t in run.tags] == g["exact_layer_tags"]
        assert layer_digest(run.layers) == g["exact_layer_digest"], name


def test_instances_bloom_treewidth_and_orders(E, goldens, gpu):
    for name, g in goldens["instances"].items():
        graph = E.Graph.parse(instance_text(name))
        res = E.solve(graph, E.Options(dedup="bloom", emit_order=True))
        assert res.kind == "exact" and res.value == g["bloom_tw"] == g["tw"]
        w, ok = graph.check_order(res.order)
        assert ok and w == g["tw"]


def test_queen6_6_mmw(E, goldens, gpu):
    graph = E.Graph.parse(instance_text("queen6_6"))
    ex = E.solve(graph, E.Options(dedup="exact", use_mmw=True))
    assert ex.stats_json == goldens["queen6_6_exact_mmw"]["stats"]
    bl = E.solve(graph, E.Options(dedup="bloom", use_mmw=True))
    ref = json.loads(goldens["queen6_6_bloom_mmw"]["stats"])
    got = json.loads(bl.stats_json)
    assert got["result"]["value"] == 25 == ref["result"]["value"]
    # absent Bloom false positives the counters are order-independent
    assert got["totals"] == ref["totals"]


def test_corpus_exact_stats(E, goldens, gpu):
    for c in goldens["corpus"]:
        rows = G.random_graph(c["seed"], c["n"], c["p"])
        res = E.solve(E.Graph.from_rows(rows), E.Options(dedup="exact", start_k=c["start_k"]))
        assert res.value == c["tw"]
        assert res.stats_json == c["exact_stats"], c["seed"]


def test_g40_exact_full_sweep(E, goldens, gpu):
    """BASELINE cfg 3 (G(40,0.3) seed 1): 3.3M expanded states, every layer
    counter identical to the reference."""
    g = goldens["g40_03"]["1"]
    res = E.solve(E.Graph.from_rows(G.random_graph(1, 40, 0.3)), E.Options(dedup="exact"))
    assert res.value == g["tw"] == 22
    assert res.stats_json == g["exact_stats"]


def test_capacity_overflow_is_a_lower_bound(E, ref, gpu):
    for seed in range(20):
        rows = G.random_graph(seed * 53 + 9, 10, 0.5)
        for cap in (2, 6):
            opts = dict(dedup="exact", max_layer_states=cap, start_k=0)
            a = E.solve(E.Graph.from_rows(rows), E.Options(**opts))
            b = ref.solve(rows, dedup="exact", cap=cap, start_k=0)
            assert (a.kind == "exact") == (b["kind"] == "exact")
            assert a.value == b["value"]
            assert a.stats_json == b["stats"]


def test_solver_matches_reference_across_option_mixes(E, ref, gpu):
    for seed in range(40):
        n = 4 + seed % 12
        rows = G.random_graph(seed * 101 + 7, n, 0.15 + 0.1 * (seed % 7))
        mixes = [dict(dedup="exact", emit_order=True),
                 dict(dedup="exact", split="none", use_clique=False, use_improvement=False,
                      emit_order=True),
                 dict(dedup="exact", split="connected", use_mmw=True, emit_order=True)]
        for m in mixes:
            a = E.solve(E.Graph.from_rows(rows), E.Options(**m))
            b = ref.solve(rows, dedup="exact", split={"none": 0, "connected": 1}.get(m.get("split"), 2),
                          mmw=m.get("use_mmw", False), clique=m.get("use_clique", True),
                          improvement=m.get("use_improvement", True), emit_order=True)
            assert a.stats_json == b["stats"], (seed, m)
        res = E.solve(E.Graph.from_rows(rows), E.Options(dedup="bloom", emit_order=True))
        w, ok = E.Graph.from_rows(rows).check_order(res.order)
        assert ok and w == res.value


def test_bloom_probe_positions_and_exactly_once(E, oracle, gpu):
    key = 0x0123456789ABCDEF  # test_bloom.cpp:46-56
    m, novel, bits = E.bloom_insert(1000, [key], want_bits=True)
    assert novel == [True]
    h1, h2 = oracle.hash_pair(key)
    expected = {(h1 + i * h2) % m for i in range(1, 18)}
    got = {w * 32 + b for w, word in enumerate(bits) for b in range(32) if word >> b & 1}
    assert got == expected
    # concurrent duplicate inserts stay exactly once (test_bloom.cpp:122-139)
    keys = [(i * 0x9E3779B97F4A7C15 + 12345) & (2**64 - 1) for i in range(5000)]
    batch = keys * 8
    random.Random(1).shuffle(batch)
    _, novel, _ = E.bloom_insert(len(keys) * 2, batch)
    per_key = {}
    for k_, nv in zip(batch, novel):
        per_key[k_] = per_key.get(k_, 0) + nv
    assert sum(novel) == len(keys)
    assert all(v == 1 for v in per_key.values())
    # same bits as the sequential reference filter
    _, seq = oracle.bloom_insert_seq(len(keys) * 2, keys)
    m2, _, bits2 = E.bloom_insert(len(keys) * 2, keys, want_bits=True)
    assert sum(bin(w).count("1") for w in bits2) > 0 and m2 > 0


def test_bloom_fp_rate_window(E, oracle, gpu):
    """Filled on the device, queried by the oracle's might_contain: the FP
    rate at the default operating point stays in the reference's acceptance
    window (acceptance.cpp:291-338): 0.3x..3x of 9.84e-6."""
    def splitmix(x):
        x = (x + 0x9E3779B97F4A7C15) & (2**64 - 1)
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & (2**64 - 1)
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & (2**64 - 1)
        return x ^ (x >> 31)
    fill = [splitmix(i) for i in range(100_000)]
    m, novel, bits = E.bloom_insert(100_000, fill, want_bits=True)
    assert all(novel[:10])
    assert oracle.bloom_query(bits, m, fill) == len(fill)  # no false negatives
    probe = [splitmix((1 << 32) + j) for j in range(1_000_000)]
    rate = oracle.bloom_query(bits, m, probe) / len(probe)
    assert 0.3 * 9.838577e-6 <= rate <= 3 * 9.838577e-6


def test_partitioned_bloom_large_filter(E, gpu):
    """Bloom mode with a filter beyond 2^28 bits takes scatter/part/append:
    exact dedup per bucket, then the reference's filter on each distinct key
    once. Same verdicts as exact mode; every layer a duplicate-free subset of
    the exact expansion of its parents; the 2^28-bit fused path (ETWG_DEBUG
    64 forces it off here) agrees on the verdicts."""
    rows = G.random_graph(1, 40, 0.3)
    for k in (21, 22):
        ex = E.decide(rows, k, dedup="exact", cap=1 << 31)
        bl = E.decide(rows, k, dedup="bloom", cap=1 << 31)
        assert bl.outcome == ex.outcome
        for layer in bl.layers:
            keys = [s for s, _ in layer]
            assert len(keys) == len(set(keys))
        first = [sorted(s for s, _ in x) for x in bl.layers]
        want = [sorted(s for s, _ in x) for x in ex.layers]
        for a, b in zip(first, want):
            if a != b:
                assert set(a) <= set(b)
                break
        # re-expanding a Bloom layer exactly contains the next Bloom layer
        for r in range(min(4, len(bl.layers) - 1)):
            nxt = E.expand_layer(rows, k, bl.layers[r], dedup="exact", cap=1 << 31)
            assert set(s for s, _ in bl.layers[r + 1]) <= set(s for s, _ in nxt.layers[0])
    g = E.Graph.from_rows(rows)
    res = E.solve(g, E.Options(dedup="bloom", max_layer_states=1 << 31))
    assert res.value == 22


def _run_with_env(env_extra, code):
    import os
    import subprocess
    import sys
    env = dict(os.environ, **env_extra)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_hash_range_passes_agree(gpu):
    """f4 (out-of-HBM child records): with ETWG_PASSES=P every exact round
    runs as P hash-range passes (K1 reruns per pass, each pass dedups and
    marks only its buckets, the append runs once). Layers, histories and
    counters are identical to the one-pass rounds, also under aborts."""
    one = _run_with_env({}, _TIGHT_CODE)
    assert one == _run_with_env({"ETWG_PASSES": "4"}, _TIGHT_CODE)
    assert one == _run_with_env({"ETWG_PASSES": "8", "ETWG_DEBUG": "1024"}, _TIGHT_CODE)
    assert one == _run_with_env({"ETWG_PASSES": "2", "ETWG_DEBUG": "8192"}, _TIGHT_CODE)


def test_global_table_equals_buckets(gpu):
    """Exact rounds of one-word keys dedup in one global open-addressing
    table (default) instead of bucket records + per-bucket shared tables
    (ETWG_GTAB=0). Both keep each key's minimum emission rank, so layers,
    histories and every counter are identical — also with undersized tables
    (ETWG_DEBUG 1024: probe-chain overflow aborts and re-runs), several
    hash-range passes, and the warp-per-parent scatter (ETWG_DEBUG 256)."""
    buckets = _run_with_env({"ETWG_GTAB": "0"}, _TIGHT_CODE)
    assert buckets == _run_with_env({}, _TIGHT_CODE)
    assert buckets == _run_with_env({"ETWG_DEBUG": "1024"}, _TIGHT_CODE)
    assert buckets == _run_with_env({"ETWG_PASSES": "4", "ETWG_DEBUG": "1024"}, _TIGHT_CODE)
    assert buckets == _run_with_env({"ETWG_DEBUG": "256"}, _TIGHT_CODE)
    assert buckets == _run_with_env({"ETWG_DEBUG": "128"}, _TIGHT_CODE)


def test_graph_replay_equals_launches(gpu):
    """Round chunks replayed from captured CUDA graphs (default) give the
    same layers, histories and counters as kernel-by-kernel launches
    (ETWG_GRAPHS=0), including rounds that abort, grow a buffer (which
    invalidates the cached graphs) and re-run."""
    eager = _run_with_env({"ETWG_GRAPHS": "0"}, _TIGHT_CODE)
    assert eager == _run_with_env({}, _TIGHT_CODE)
    assert eager == _run_with_env({"ETWG_DEBUG": "1024"}, _TIGHT_CODE)


def _run_with_debug(flags, code):
    """Runs `code` in a fresh interpreter with ETWG_DEBUG=flags (the engine
    reads it when a decide starts) and returns its JSON output."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, ETWG_DEBUG=str(flags))
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


_MODES_CODE = """
import json, sys
sys.path.insert(0, ".")
from paper_1709_09990_b200 import elimtw as E, generators as G
res = {}
for name, rows, k, mmw in (("q", G.queen_graph(5, 5), 18, True), ("g", G.random_graph(4, 30, 0.3), 14, True),
                           ("x", G.random_graph(1, 40, 0.3), 21, False), ("w", G.random_graph(9, 70, 0.07), 5, False)):
    # Bloom only where it runs through the scatter (MMW decides); the fused
    # Bloom kernel's layers depend on insertion order like the reference's
    for dedup in ("exact", "bloom") if mmw else ("exact",):
        r = E.decide(rows, k, dedup=dedup, mmw=mmw, rounds=8 if name == "w" else -1)
        res[name + dedup] = [r.outcome, [x.tuple() for x in r.rounds], r.layers if dedup == "exact" else
                             [sorted(s for s, _ in l) for l in r.layers]]
print(json.dumps(res))
"""


def test_scatter_thread_and_warp_modes_agree(gpu):
    """The scatter's one-thread-per-parent mode (large layers) and its
    warp-per-parent mode (small layers) give identical exact layers, orders,
    histories and counters — with and without MMW, 64- and 128-bit keys."""
    thread = _run_with_debug(128, _MODES_CODE)
    warp = _run_with_debug(256, _MODES_CODE)
    assert thread == warp


_TIGHT_CODE = """
import json, sys
sys.path.insert(0, ".")
from paper_1709_09990_b200 import elimtw as E, generators as G
res = {}
for name, rows, k, mmw in (("g", G.random_graph(1, 40, 0.3), 21, False), ("q", G.queen_graph(5, 5), 18, True),
                           ("w", G.random_graph(9, 70, 0.07), 5, False)):
    r = E.decide(rows, k, dedup="exact", mmw=mmw, rounds=8 if name == "w" else -1)
    res[name] = [r.outcome, r.witness_set, r.witness_hist, [x.tuple() for x in r.rounds], r.layers]
print(json.dumps(res))
"""


def test_partitioned_rounds_survive_aborts(gpu):
    """Undersized bucket plans (ETWG_DEBUG 1024: 1/16 of the partitions, 1/4
    of the record capacity) make rounds abort and re-run with raised floors;
    exact layers, orders, histories and counters are unchanged."""
    assert _run_with_debug(1024, _TIGHT_CODE) == _run_with_debug(0, _TIGHT_CODE)


def test_compact_and_wide_records_agree(gpu):
    """ETWG_DEBUG 8192 turns on the 8-byte {mixed-key bits, parent} records
    for rounds of one-word keys (PartPlan, wavefront.cu; the default is the
    16-byte {key, rank} record). Layers, histories and counters must not
    depend on the format, including under the tight plans' aborts."""
    wide = _run_with_debug(0, _TIGHT_CODE)
    assert wide == _run_with_debug(8192, _TIGHT_CODE)
    assert wide == _run_with_debug(1024 | 8192, _TIGHT_CODE)
