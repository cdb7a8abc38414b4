import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_1709_09990_b200 import elimtw as E, generators as G
from checkers import Oracle
o = Oracle()
nbad = 0
for rep in range(3):
  for seed in range(30):
    n = 6 + seed % 18
    rows = G.random_graph(seed * 17 + 3, n, 0.2 + 0.04 * (seed % 6))
    for k in (n // 4, n // 3):
        a = E.decide(rows, k, dedup="bloom")
        b = o.decide(rows, k, dedup="bloom")
        for li, (la, lb) in enumerate(zip(a.layers, b.layers)):
            sa, sb = set(s for s, _ in la), set(s for s, _ in lb)
            if sa != sb or len(la) != len(sa):
                nbad += 1
                if nbad <= 4:
                    print("rep", rep, "seed", seed, "n", n, "k", k, "layer", li, "dev", len(la), len(sa), "orc", len(lb))
                    print("  dev rounds", [x.tuple()[2:5] for x in a.rounds][:li+2])
                    print("  orc rounds", [x.tuple()[2:5] for x in b.rounds][:li+2])
                    print("  missing", [hex(x) for x in sorted(sb - sa)][:5], "extra", [hex(x) for x in sorted(sa - sb)][:5])
                    # was the missing key's parent present in previous layer on device?
                    if li > 0:
                        prev = set(s for s, _ in a.layers[li-1])
                        for x in sorted(sb - sa)[:3]:
                            parents = [x & ~(1 << v) for v in range(n) if (x >> v) & 1]
                            print("   parents in dev prev layer:", [hex(p) for p in parents if p in prev])
                break
print("bad", nbad)
