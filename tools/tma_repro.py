import sys, os
sys.path.insert(0, '.')
from paper_1709_09990_b200 import elimtw as E, generators as G
which = sys.argv[1]
if which == "expand":
    rows = G.random_graph(100, 10, 0.3)
    r = E.expand_layer(rows, 4, [(0, 0xFFFFFFFF)], dedup="exact")
    print("expand ok", r.rounds[0].emitted, flush=True)
else:
    rows = G.random_graph(5, 4, 0.15)
    r = E.decide(rows, 1, dedup="exact", cap=5)
    print("decide ok", [x.emitted for x in r.rounds], flush=True)
