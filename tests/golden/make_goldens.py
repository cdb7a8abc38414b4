"""Regenerates tests/golden/goldens.json from the UNMODIFIED reference.

Run in the dev container (needs oracle/_ref/libetwref.so, built from
/root/reference sources by `make -C oracle ref`):

    python tests/golden/make_goldens.py

Every value below comes out of the reference's own code paths (decide,
solve + stats_json, Murmur3 / ConcurrentBloom, MMW, preprocess) through
oracle/ref_harness.cpp; the instance files in tests/golden/instances/ are the
reference's test instances (proj/tests/instances/*.gr), kept as data.
"""
from __future__ import annotations

import hashlib
import json
import os
import struct
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from checkers import RefLib  # noqa: E402
from paper_1709_09990_b200 import generators as G  # noqa: E402

INSTANCES = ["water", "myciel4", "McGeeGraph", "queen5_5", "queen6_6"]


def layer_digest(layers) -> str:
    """sha256 over every layer in order: u32 size, then (u64 set, u32 hist)
    per state in layer order (sets > 64 bits use two u64 words)."""
    h = hashlib.sha256()
    for layer in layers:
        h.update(struct.pack("<I", len(layer)))
        for s, hist in layer:
            h.update(struct.pack("<QQI", s & (2**64 - 1), s >> 64, hist))
    return h.hexdigest()


def main() -> None:
    ref = RefLib()
    out = {"generated_by": "tests/golden/make_goldens.py (reference elimtw via oracle/_ref)"}

    # Murmur3 published vectors (proj/tests/test_bloom.cpp:20-34)
    vec = [("", 0), ("", 1), ("", 0xFFFFFFFF), ("\0\0\0\0", 0), ("a", 0x9747B28C),
           ("aa", 0x9747B28C), ("aaa", 0x9747B28C), ("aaaa", 0x9747B28C), ("ab", 0x9747B28C),
           ("abc", 0x9747B28C), ("abcd", 0x9747B28C), ("Hello, world!", 0x9747B28C)]
    out["murmur3"] = [[d.encode("latin1").hex(), seed, ref.murmur3(d.encode("latin1"), seed)]
                      for d, seed in vec]
    keys = [0, 1, 7, 0x0123456789ABCDEF, 2**64 - 1, 2**63, 0xDEADBEEF, 3 << 40]
    out["hash_pair"] = [[k, *ref.hash_pair(k)] for k in keys]
    # sequential bloom novelty on a dup-heavy stream (bloom.cpp:86-97)
    stream = [(i * 0x9E3779B97F4A7C15) & (2**64 - 1) for i in range(3000)]
    stream += stream[::7]
    m, novel = ref.bloom_insert_seq(1000, stream)
    out["bloom_seq"] = {"expected": 1000, "m": m, "novel_count": sum(novel),
                        "novel_digest": hashlib.sha256(bytes(novel)).hexdigest()}
    out["bloom_fp"] = {"1e6@1e6": ref.bloom_expected_fp(1_000_000, 1_000_000),
                       "2e6@1e6": ref.bloom_expected_fp(1_000_000, 2_000_000)}

    # instances: tw and the full stats report in exact mode (byte target)
    inst = {}
    for name in INSTANCES:
        text = open(os.path.join(HERE, "instances", name + ".gr")).read()
        rows = ref.parse(text)
        ex = ref.solve(rows, dedup="exact", emit_order=True)
        bl = ref.solve(rows, dedup="bloom")
        entry = {"n": len(rows), "tw": ex["value"], "exact_stats": ex["stats"],
                 "exact_order": ex["order"], "bloom_tw": bl["value"],
                 "max_clique": ref.max_clique(rows), "mmw_root": ref.mmw_lower_bound(rows)}
        run = ref.solve_layers(rows)
        entry["exact_layer_digest"] = layer_digest(run.layers)
        entry["exact_layer_sizes"] = [len(x) for x in run.layers]
        entry["exact_layer_tags"] = [[r.k, r.round] for r in run.rounds]
        inst[name] = entry
    out["instances"] = inst

    # MMW on queen6_6 with Bloom (BASELINE cfg 2), counters of the 1-thread run
    rows = ref.parse(open(os.path.join(HERE, "instances", "queen6_6.gr")).read())
    q = ref.solve(rows, dedup="bloom", mmw=True)
    out["queen6_6_bloom_mmw"] = {"tw": q["value"], "stats": q["stats"]}
    q = ref.solve(rows, dedup="exact", mmw=True)
    out["queen6_6_exact_mmw"] = {"tw": q["value"], "stats": q["stats"]}

    # random corpus: treewidth + full exact stats (helpers.hpp random_graph)
    corpus = []
    for seed in range(40):
        n = 6 + seed % 12
        p = 0.2 + 0.05 * (seed % 7)
        rows = G.random_graph(seed * 977 + 13, n, p)
        ex = ref.solve(rows, dedup="exact", start_k=0 if seed % 3 == 0 else -1)
        corpus.append({"seed": seed * 977 + 13, "n": n, "p": p, "start_k": 0 if seed % 3 == 0 else -1,
                       "tw": ex["value"], "exact_stats": ex["stats"]})
    out["corpus"] = corpus

    # G(40, 0.3) seeds 1, 2 (BASELINE cfg 3): tw and totals
    big = {}
    for seed in (1,):
        rows = G.random_graph(seed, 40, 0.3)
        ex = ref.solve(rows, dedup="exact")
        big[str(seed)] = {"tw": ex["value"], "exact_stats": ex["stats"]}
    out["g40_03"] = big

    with open(os.path.join(HERE, "goldens.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("wrote", os.path.join(HERE, "goldens.json"))


if __name__ == "__main__":
    main()
