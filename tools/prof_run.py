"""Profiling driver (not a benchmark): runs the bench workload a few times so
ncu can capture launches. Usage: python tools/prof_run.py [reps] [dedup]"""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1709_09990_b200 import elimtw as E, generators as G
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
dedup = sys.argv[2] if len(sys.argv) > 2 else "bloom"
g = E.Graph.from_rows(G.random_graph(1, 40, 0.3))
for _ in range(reps):
    r = E.solve(g, E.Options(dedup=dedup))
print("tw", r.value)
