import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_1709_09990_b200 import elimtw as E, generators as G
from checkers import Oracle
o = Oracle()
seed, k = 12, 4
n = 6 + seed % 18
rows = G.random_graph(seed * 17 + 3, n, 0.2 + 0.04 * (seed % 6))
b = o.decide(rows, k, dedup="bloom", keep_layers=False)
want = [x.emitted for x in b.rounds]
bad = 0
for rep in range(300):
    a = E.decide(rows, k, dedup="bloom", keep_layers=False)
    if [x.emitted for x in a.rounds] != want:
        bad += 1
print("flags", os.environ.get("ETWG_DEBUG"), "bad", bad, "of 300")
