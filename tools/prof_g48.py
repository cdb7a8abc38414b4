"""Profiling driver (not a benchmark): G(48,0.2) full sweep with per-kernel
event timing. Usage: python tools/prof_g48.py [dedup] [cap]"""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1709_09990_b200 import elimtw as E, generators as G
dedup = sys.argv[1] if len(sys.argv) > 1 else "exact"
cap = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 31
n = int(os.environ.get("PROBE_N", "48")); p = float(os.environ.get("PROBE_P", "0.2"))
g = E.Graph.from_rows(G.random_graph(1, n, p))
E.solve(g, E.Options(dedup=dedup, max_layer_states=cap))  # warm (allocations)
E.set_profiling(True); E.reset_times()
t0 = time.perf_counter()
r = E.solve(g, E.Options(dedup=dedup, max_layer_states=cap))
dt = time.perf_counter() - t0
print(dedup, "tw", r.value, f"{dt:.3f}s (profiled, serialised)")
print(json.dumps(E.times(), indent=1))
