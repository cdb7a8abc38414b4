import sys, os, random
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_1709_09990_b200 import elimtw as E, generators as G
from checkers import Oracle
o = Oracle()
def norm(r): return (r.outcome, r.witness_set, r.witness_hist, r.overflowed, [x.tuple() for x in r.rounds], r.layers)
def wide(tag):
    bad = 0
    for i, n in enumerate((66, 72)):
        rows = G.random_graph(i + 7, n, 8.0 / n)
        for dedup in ("exact", "bloom"):
            a = E.decide(rows, 5, dedup=dedup, rounds=6)
            b = o.decide(rows, 5, dedup=dedup, rounds=6)
            if dedup == "exact" and norm(a) != norm(b):
                bad += 1
                print(tag, "MISMATCH n", n, hex(a.witness_set), hex(b.witness_set), [x.emitted for x in a.rounds], [len(l) for l in a.layers])
                for li,(la,lb) in enumerate(zip(a.layers,b.layers)):
                    if la!=lb: print("   layer", li, "sorted eq", sorted(la)==sorted(lb), la[:2], lb[:2]); break
    print(tag, "bad", bad)
wide("fresh")
# what the suite runs before: small exact decides with/without mmw and caps
for seed in range(60):
    n = 4 + seed % 22
    rows = G.random_graph(seed * 131 + 5, n, 0.15 + 0.05 * (seed % 8))
    for k in sorted({max(0, n // 4), n // 3}):
        cap = 5 if seed % 7 == 0 else 10_000_000
        E.decide(rows, k, dedup="exact", cap=cap)
wide("after-exact")
for seed in range(30):
    n = 6 + seed % 18
    rows = G.random_graph(seed * 17 + 3, n, 0.2 + 0.04 * (seed % 6))
    for k in (n // 4, n // 3):
        E.decide(rows, k, dedup="bloom")
wide("after-bloom")
