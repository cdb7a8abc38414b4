"""Reference goldens for the large BASELINE configs (TEST INFRASTRUCTURE ONLY).

Every value comes out of the UNMODIFIED reference (oracle/_ref/libetwref.so,
built from /root/reference/proj/src by `make -C oracle ref`) through its own
`solve()` (proj/src/solver.cpp:149-196) and `stats_json` (solver.cpp:198-297).

    python tests/golden/make_big_goldens.py small
        G(40,0.3) seed 2 (cfg 3, 8,261,454 expanded), myciel4 exact with and
        without MMW (acceptance criterion 4, proj/tests/acceptance.cpp:245-286).
        Runs in minutes here.

    python tests/golden/make_big_goldens.py g48 [threads]
        G(48,0.2) seed 1 (cfg 4, the bench workload), exact dedup,
        max_layer_states = 2^31, full k sweep. Its largest round holds ~1.8e9
        child entries of 24 B in the reference's thread-local vectors plus the
        concatenated copy (dp.cpp:118-135), which does not fit this container's
        62 GB, so it runs on the GPU box's host (the prebuilt .so travels; the
        reference tree is not read there). Output: tests/golden/g48_ref.json.

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


def g48(threads: int) -> None:
    ref = RefLib()
    rows = G.random_graph(1, 48, 0.2)
    t = time.time()
    ex = ref.solve(rows, dedup="exact", threads=threads, cap=BIG_CAP, json_len=1 << 26)
    wall = time.time() - t
    tot = _totals(ex["stats"])
    out = {"generated_by": "tests/golden/make_big_goldens.py g48 (reference elimtw via oracle/_ref)",
           "graph": "random_graph(seed=1, n=48, p=0.2)", "options": {
               "dedup": "exact", "max_layer_states": BIG_CAP, "threads": threads,
               "emit_order": False},
           "tw": ex["value"], "kind": ex["kind"], "exact_stats": ex["stats"],
           "ref_wall_s": round(wall, 1), "host": _host(), "totals": tot}
    path = os.path.join(HERE, "g48_ref.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("wrote", path, "tw", ex["value"], "wall", round(wall, 1), "s", tot)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "small"
    if what == "small":
        small()
    elif what == "g48":
        g48(int(sys.argv[2]) if len(sys.argv) > 2 else (os.cpu_count() or 1))
    else:
        raise SystemExit(f"unknown target {what}")
