"""Dump the device solve's stats JSON for G(48,0.2) seed 1 (BASELINE cfg 4,
the bench workload) with the options tests/golden/make_big_goldens.py g48
uses, plus each round's offered-children count (emitted + duplicates), so it
can be compared with the reference golden byte for byte.
Usage: python tools/g48_stats.py THREADS OUT.json"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1709_09990_b200 import elimtw as E, generators as G  # noqa: E402

threads = int(sys.argv[1])
out = sys.argv[2]
g = E.Graph.from_rows(G.random_graph(1, 48, 0.2))
t = time.perf_counter()
r = E.solve(g, E.Options(dedup="exact", max_layer_states=1 << 31, thread_count=threads))
dt = time.perf_counter() - t
st = json.loads(r.stats_json)
peak = max((l["emitted"] + l["duplicates"], a["k"], l["round"])
           for c in st["components"] for a in c["attempts"] for l in a["layers"])
json.dump({"tw": r.value, "kind": r.kind, "stats": r.stats_json, "s": dt,
           "peak_offered": peak}, open(out, "w"))
print("tw", r.value, "s", round(dt, 3), "peak offered (n, k, round)", peak)
