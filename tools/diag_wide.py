import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_1709_09990_b200 import elimtw as E, generators as G
from checkers import Oracle
o = Oracle()
for i, n in enumerate((66, 72, 80, 96, 112, 128)):
    rows = G.random_graph(i + 7, n, 8.0 / n)
    for dedup in ("exact",):
        a = E.decide(rows, 5, dedup=dedup, rounds=6)
        b = o.decide(rows, 5, dedup=dedup, rounds=6)
        print(n, dedup, a.outcome, b.outcome, hex(a.witness_set), hex(b.witness_set), hex(a.witness_hist), hex(b.witness_hist))
        print("  dev", [x.tuple()[2:] for x in a.rounds])
        print("  orc", [x.tuple()[2:] for x in b.rounds])
        for li, (la, lb) in enumerate(zip(a.layers, b.layers)):
            if la != lb:
                print("  layer", li, len(la), len(lb), "sorted eq", sorted(la) == sorted(lb))
                for j, (x, y) in enumerate(zip(la, lb)):
                    if x != y:
                        print("   first diff", j, [(hex(s), hex(h)) for s, h in la[j:j+3]], [(hex(s), hex(h)) for s, h in lb[j:j+3]]); break
                break
        print("  last layer dev front", [hex(s) for s,_ in a.layers[-1][:3]] if a.layers else None)
