"""Bloom vs exact on the bench graph, round by round (not a benchmark):
solves G(48,0.2) seed 1 in both modes (max_layer_states 2^31), writes both
stats JSONs and prints every round whose counters differ.
Usage: python tools/bloom_diff.py OUT_PREFIX"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1709_09990_b200 import elimtw as E, generators as G  # noqa: E402

pre = sys.argv[1]
g = E.Graph.from_rows(G.random_graph(1, 48, 0.2))
st = {}
for mode in ("exact", "bloom"):
    r = E.solve(g, E.Options(dedup=mode, max_layer_states=1 << 31))
    st[mode] = json.loads(r.stats_json)
    with open(f"{pre}_{mode}.json", "w") as f:
        f.write(r.stats_json)
ex = {(a["k"], l["round"]): l for c in st["exact"]["components"] for a in c["attempts"] for l in a["layers"]}
bl = {(a["k"], l["round"]): l for c in st["bloom"]["components"] for a in c["attempts"] for l in a["layers"]}
for key in sorted(set(ex) | set(bl)):
    a, b = ex.get(key), bl.get(key)
    if a is None or b is None or (a["expanded"], a["emitted"]) != (b["expanded"], b["emitted"]):
        print("k=%d round=%d" % key, "exact", a and (a["expanded"], a["emitted"], a["duplicates"]),
              "bloom", b and (b["expanded"], b["emitted"], b["duplicates"]))
