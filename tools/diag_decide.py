"""Debug helper: first divergence between device decide and the oracle."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_1709_09990_b200 import elimtw as E, generators as G
from checkers import Oracle
o = Oracle()
cases = [(5, 2), (5, 3)]
for seed, k in cases:
    n = 4 + seed % 30
    rows = G.random_graph(seed * 131 + 5, n, 0.15 + 0.05 * (seed % 8))
    a = E.decide(rows, k, dedup="exact")
    b = o.decide(rows, k, dedup="exact")
    print("case", seed, k, "n", n, a.outcome, b.outcome)
    print(" dev rounds", [x.tuple() for x in a.rounds])
    print(" orc rounds", [x.tuple() for x in b.rounds])
    for li, (la, lb) in enumerate(zip(a.layers, b.layers)):
        if la != lb:
            print(" layer", li, "len", len(la), len(lb))
            print("  sorted sets equal:", sorted(s for s,_ in la) == sorted(s for s,_ in lb))
            for j, (x, y) in enumerate(zip(la, lb)):
                if x != y:
                    print("  first diff at", j, [(hex(s), hex(h)) for s,h in la[max(0,j-2):j+4]], "vs", [(hex(s), hex(h)) for s,h in lb[max(0,j-2):j+4]])
                    break
            break
