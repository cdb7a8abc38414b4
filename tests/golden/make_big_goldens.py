"""Reference goldens for the large BASELINE configs (TEST INFRASTRUCTURE ONLY).

Every value comes out of the UNMODIFIED reference (oracle/_ref/libetwref.so,
built from /root/reference/proj/src by `make -C oracle ref`) through its own
`solve()` (proj/src/solver.cpp:149-196) and `stats_json` (solver.cpp:198-297).

    python tests/golden/make_big_goldens.py small
        G(40,0.3) seed 2 (cfg 3, 8,261,454 expanded), myciel4 exact with and
        without MMW (acceptance criterion 4, proj/tests/acceptance.cpp:245-286).
        Runs in minutes here.

    python tests/golden/make_big_goldens.py g48 THREADS K [K ...]
        G(48,0.2) seed 1 (cfg 4, the bench workload), exact dedup,
        max_layer_states = 2^31: the reference's decide (dp.cpp:167-194) on
        the attempts solve() makes (solver.cpp:21-67: the largest biconnected
        block, the forbidden max clique, the improved graph per k), one JSON
        per run: tests/golden/g48_ref_k<K..>.json with every round's
        LayerStats and the outcome. The k = 24 attempt alone offers 9.4e9
        children (1.86e9 in one round, 24 B each in the reference's
        thread-local vectors plus the concatenated copy, dp.cpp:118-135): it
        needs ~140 GB and ~30 min of the reference's single-threaded sorts, so
        the sweep runs on the GPU box's host (16 cores, 196 GB) in pieces that
        fit a call; the prebuilt .so travels, the reference tree is not read
        there.

    python tests/golden/make_big_goldens.py queen88
        queen8_8 (n = 64, tw 45) exact with the order, ~6 min on 8 cores.

    python tests/golden/make_big_goldens.py grid88
        8x8 grid + 6 chords (n = 64, default cap: overflow -> lower bound),
        ~20 min on 8 cores.

    python tests/golden/make_big_goldens.py wide72
        G(72,0.5) seed 1 on the 128-bit path (oracle checker; no reference
        above 64 vertices).

    python tests/golden/make_big_goldens.py g48-merge
        Merges the pieces and the cheap solve() prelude computed here (block,
        clique, MMW bound, start k, improvement edges per k) into
        tests/golden/g48_ref.json.

The outputs are committed next to this script.
"""
from __future__ import annotations

import json
import os
import platform
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from checkers import RefLib  # noqa: E402
from paper_1709_09990_b200 import generators as G  # noqa: E402

BIG_CAP = 1 << 31


def _host() -> dict:
    mem = 0
    try:
        with open("/proc/meminfo") as f:
            mem = int(f.readline().split()[1]) // (1 << 20)
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "mem_gb": mem, "machine": platform.machine()}


def _totals(stats: str) -> dict:
    js = json.loads(stats)
    return js.get("totals", {})


def small() -> None:
    ref = RefLib()
    out = {"generated_by": "tests/golden/make_big_goldens.py small (reference elimtw via oracle/_ref)"}
    rows = G.random_graph(2, 40, 0.3)
    t = time.time()
    ex = ref.solve(rows, dedup="exact", threads=os.cpu_count())
    out["g40_03_seed2"] = {"tw": ex["value"], "kind": ex["kind"], "threads": os.cpu_count(),
                           "exact_stats": ex["stats"], "ref_s": round(time.time() - t, 3)}
    text = open(os.path.join(HERE, "instances", "myciel4.gr")).read()
    rows = ref.parse(text)
    plain = ref.solve(rows, dedup="exact", emit_order=True)
    mmw = ref.solve(rows, dedup="exact", mmw=True, emit_order=True)
    out["myciel4_exact_mmw"] = {"tw": mmw["value"], "order": mmw["order"],
                                "stats": mmw["stats"], "plain_tw": plain["value"],
                                "plain_stats": plain["stats"]}
    path = os.path.join(HERE, "big_goldens.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("wrote", path)


def queen88() -> None:
    """queen8_8 (n = 64: the full 64-bit word; tw 45), exact
    dedup with max_layer_states 2^31 (the default 10M would overflow), with
    the elimination order: merged into big_goldens.json."""
    ref = RefLib()
    rows = G.queen_graph(8, 8)
    t = time.time()
    ex = ref.solve(rows, dedup="exact", threads=os.cpu_count(), cap=BIG_CAP, emit_order=True,
                   json_len=1 << 26)
    path = os.path.join(HERE, "big_goldens.json")
    out = json.load(open(path))
    out["queen8_8"] = {"tw": ex["value"], "kind": ex["kind"], "threads": os.cpu_count(),
                       "max_layer_states": BIG_CAP, "order": ex["order"], "exact_stats": ex["stats"],
                       "ref_s": round(time.time() - t, 1)}
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("queen8_8 tw", ex["value"], "in", round(time.time() - t, 1), "s")


def grid88() -> None:
    """BASELINE cfg 5a: 8x8 grid + 6 chords (seed 7), n = 64 on the one-word
    path, exact dedup with the reference's default 10M layer cap: the layers
    overflow (truncation to the lowest emission ranks, dp.cpp:152-155) and the
    solve returns the lower bound. Merged into big_goldens.json."""
    ref = RefLib()
    rows = G.grid_with_chords(8, 8, 6, 7)
    t = time.time()
    ex = ref.solve(rows, dedup="exact", threads=os.cpu_count(), json_len=1 << 26)
    path = os.path.join(HERE, "big_goldens.json")
    out = json.load(open(path))
    out["grid8x8_chords6_seed7"] = {"tw": ex["value"], "kind": ex["kind"], "threads": os.cpu_count(),
                                    "exact_stats": ex["stats"], "ref_s": round(time.time() - t, 1)}
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("grid 8x8+6", ex["kind"], ex["value"], "in", round(time.time() - t, 1), "s")


def wide72() -> None:
    """BASELINE cfg 5b, the 128-bit path to an exact treewidth: G(72,0.5)
    seed 1 (tw 57, ~7.4M expanded states). No reference exists above 64
    vertices (graph.cpp:111-113), so the checker is the oracle's decide
    (oracle/etw_oracle.c, 128-bit sets) on every attempt solve() makes:
    the block, the forbidden max clique and the improved graph per k come
    from the host preprocessing (tested against the reference by embedding,
    tests/test_host.py). Merged into big_goldens.json."""
    from checkers import Oracle
    from paper_1709_09990_b200 import elimtw as E
    oracle = Oracle()
    rows = G.random_graph(1, 72, 0.5)
    blocks = E.split(rows)
    verts = max(blocks, key=lambda b: len(b[0]))[0]
    sub = [sum(1 << j for j, u in enumerate(verts) if rows[v] >> u & 1) for v in verts]
    clique = E.max_clique(sub)
    k = max(bin(clique).count("1") - 1, E.mmw_lower_bound(sub))
    attempts = []
    t = time.time()
    while True:
        gk = E.improve_graph(sub, k)
        run = oracle.decide(gk, k, forbidden=clique, dedup="exact", cap=BIG_CAP, keep_layers=False)
        attempts.append({"k": k, "outcome": run.outcome, "witness": [run.witness_set & (2**64 - 1),
                                                                     run.witness_set >> 64],
                         "layers": [[x.round, x.expanded, x.emitted, x.duplicates, x.mmw_pruned,
                                     bool(x.overflowed)] for x in run.rounds]})
        print("k", k, run.outcome, sum(x.expanded for x in run.rounds), flush=True)
        if run.outcome == "feasible":
            break
        k += 1
    path = os.path.join(HERE, "big_goldens.json")
    out = json.load(open(path))
    out["g72_05_seed1"] = {"checker": "oracle decide per attempt (128-bit)", "block": verts,
                           "clique": [clique & (2**64 - 1), clique >> 64], "tw": k,
                           "attempts": attempts, "oracle_s": round(time.time() - t, 1)}
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("G(72,0.5) tw", k, "in", round(time.time() - t, 1), "s")


def _g48_block(ref):
    rows = G.random_graph(1, 48, 0.2)
    blocks = ref.split(rows, 2)
    verts = max(blocks, key=lambda b: len(b[0]))[0]
    idx = {v: i for i, v in enumerate(verts)}
    sub = []
    for v in verts:
        r = 0
        for u in range(len(rows)):
            if rows[v] >> u & 1 and u in idx:
                r |= 1 << idx[u]
        sub.append(r)
    return rows, verts, sub


def g48(threads: int, ks) -> None:
    ref = RefLib()
    _, _, sub = _g48_block(ref)
    clique = ref.max_clique(sub)
    out = {"generated_by": "tests/golden/make_big_goldens.py g48 (reference decide via oracle/_ref)",
           "threads": threads, "host": _host(), "attempts": []}
    for k in ks:
        gk = ref.improve_graph(sub, k)
        t = time.time()
        run = ref.decide(gk, k, forbidden=clique, dedup="exact", cap=BIG_CAP, threads=threads,
                         keep_layers=False)
        dt = time.time() - t
        out["attempts"].append({"k": k, "outcome": run.outcome, "overflowed": run.overflowed,
                                "witness": run.witness_set, "ref_s": round(dt, 1),
                                "layers": [[x.round, x.expanded, x.emitted, x.duplicates,
                                            x.mmw_pruned, bool(x.overflowed)] for x in run.rounds]})
        print("k", k, run.outcome, "expanded", sum(x.expanded for x in run.rounds), "s", round(dt, 1),
              flush=True)
        path = os.path.join(HERE, "g48_ref_k" + "_".join(map(str, ks)) + ".json")
        with open(path, "w") as f:
            json.dump(out, f, indent=1)


def g48_merge() -> None:
    ref = RefLib()
    rows, verts, sub = _g48_block(ref)
    clique = ref.max_clique(sub)
    mmw = ref.mmw_lower_bound(sub)
    start = max(bin(clique).count("1") - 1, mmw)
    edges = sum(bin(r).count("1") for r in sub) // 2
    attempts = {}
    pieces = []
    for name in sorted(os.listdir(HERE)):
        if name.startswith("g48_ref_k") and name.endswith(".json"):
            piece = json.load(open(os.path.join(HERE, name)))
            pieces.append({"file": name, "threads": piece["threads"], "host": piece["host"]})
            for a in piece["attempts"]:
                gk = ref.improve_graph(sub, a["k"])
                a["added_edges"] = sum(bin(r).count("1") for r in gk) // 2 - edges
                attempts[a["k"]] = a
    ks = sorted(attempts)
    assert ks == list(range(start, ks[-1] + 1)), ks
    assert all(attempts[k]["outcome"] == "infeasible" for k in ks[:-1])
    assert attempts[ks[-1]]["outcome"] == "feasible"
    out = {"generated_by": "tests/golden/make_big_goldens.py g48-merge (reference via oracle/_ref)",
           "graph": "random_graph(seed=1, n=48, p=0.2)", "max_layer_states": BIG_CAP,
           "block": verts, "clique_size": bin(clique).count("1"), "mmw_bound": mmw,
           "start_k": start, "tw": ks[-1], "attempts": [attempts[k] for k in ks],
           "expanded": sum(l[1] for k in ks for l in attempts[k]["layers"]), "pieces": pieces}
    with open(os.path.join(HERE, "g48_ref.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("tw", out["tw"], "expanded", out["expanded"])


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "small"
    if what == "small":
        small()
    elif what == "g48":
        g48(int(sys.argv[2]), [int(x) for x in sys.argv[3:]])
    elif what == "g48-merge":
        g48_merge()
    elif what == "queen88":
        queen88()
    elif what == "grid88":
        grid88()
    elif what == "wide72":
        wide72()
    else:
        raise SystemExit(f"unknown target {what}")
