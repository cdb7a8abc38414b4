import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_1709_09990_b200 import elimtw as E, generators as G
from checkers import Oracle
o = Oracle()
seed, k = 12, 4
n = 6 + seed % 18
rows = G.random_graph(seed * 17 + 3, n, 0.2 + 0.04 * (seed % 6))
b = o.decide(rows, k, dedup="bloom", keep_layers=True)
want = [x.tuple()[2:5] for x in b.rounds]
print("orc", want)
shown = 0
for rep in range(60):
    a = E.decide(rows, k, dedup="bloom", keep_layers=(rep % 2 == 0))
    got = [x.tuple()[2:5] for x in a.rounds]
    if got != want and shown < 4:
        shown += 1
        print("rep", rep, "keep", rep % 2 == 0, "dev", got)
        if a.layers:
            for li, (la, lb) in enumerate(zip(a.layers, b.layers)):
                sa, sb = set(s for s,_ in la), set(s for s,_ in lb)
                if sa != sb:
                    print("  layer", li, "missing", [hex(x) for x in sorted(sb-sa)], "extra", [hex(x) for x in sorted(sa-sb)], "dups-in-layer", len(la)-len(sa)); break
b2 = o.decide(rows, k, dedup="exact", keep_layers=False)
bad = 0
for rep in range(60):
    a = E.decide(rows, k, dedup="exact", keep_layers=False)
    if [x.tuple() for x in a.rounds] != [x.tuple() for x in b2.rounds]: bad += 1
print("exact bad", bad)
