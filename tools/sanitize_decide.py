"""Small decides for compute-sanitizer (racecheck / memcheck / synccheck) on
the lock-free kernels: exact and Bloom dedup on G(40,0.3) k=22 (the
look-back scan, shared claim tables, Bloom claim CAS), a 128-bit decide, and
a 2-virtual-shard decide (route / owner / marks).
Usage: python tools/sanitize_decide.py [exact|bloom|wide|shard2]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1709_09990_b200 import elimtw as E, generators as G  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "exact"
n = int(os.environ.get("SAN_N", "40"))
rows = G.random_graph(1, n, 0.3)
k = int(os.environ.get("SAN_K", "22"))
if mode == "wide":
    rows = G.random_graph(3, 70, 0.5)
    r = E.decide(rows, 60, dedup="exact", rounds=6)
elif mode == "shard2":
    E.set_virtual_shards(2)
    E.set_shard_handoff(0)
    r = E.decide(rows, k, dedup="exact")
else:
    r = E.decide(rows, k, dedup=mode)
print(mode, r.outcome, [x.emitted for x in r.rounds][-4:])
