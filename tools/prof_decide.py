"""Profiling driver (not a benchmark): one device decide on G(n,p) seed 1 at
a fixed k, no layer copies. Usage: python tools/prof_decide.py k dedup [reps]"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1709_09990_b200 import elimtw as E, generators as G
k = int(sys.argv[1]); dedup = sys.argv[2]; reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
n = int(os.environ.get("PROBE_N", "48")); p = float(os.environ.get("PROBE_P", "0.2"))
rows = G.random_graph(1, n, p)
if int(os.environ.get("VSHARDS", "1")) > 1:
    E.set_virtual_shards(int(os.environ["VSHARDS"]))
for _ in range(reps):
    t0 = time.perf_counter()
    r = E.decide(rows, k, dedup=dedup, cap=1 << 31, keep_layers=False)
    dt = time.perf_counter() - t0
    ex = sum(s.expanded for s in r.rounds)
    print(dedup, "k", k, r.outcome, f"{dt:.3f}s", "expanded", ex, f"{ex/dt:.3e}/s",
          "max layer", max(s.emitted for s in r.rounds), flush=True)
for s in r.rounds:
    print(s.round, s.expanded, s.emitted, s.duplicates)
