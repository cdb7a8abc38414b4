"""Probe (not a benchmark): sizes of the G(48,0.2) workload (BASELINE cfg 4)
on the device. Prints per-k totals, wall time and throughput for each dedup
mode. Usage: python tools/probe_g48.py [cap] [modes]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1709_09990_b200 import elimtw as E, generators as G  # noqa: E402

cap = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 31
modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["bloom", "exact"]
n = int(os.environ.get("PROBE_N", "48"))
p = float(os.environ.get("PROBE_P", "0.2"))
rows = G.random_graph(1, n, p)
g = E.Graph.from_rows(rows)
print("n", g.vertex_count, "m", g.edge_count, flush=True)
for mode in modes:
    t0 = time.perf_counter()
    r = E.solve(g, E.Options(dedup=mode, max_layer_states=cap))
    dt = time.perf_counter() - t0
    st = json.loads(r.stats_json)
    tot = st["totals"]
    print(mode, "tw", r.value, "kind", r.kind, f"{dt:.2f}s", "expanded", tot["expanded"],
          f"{tot['expanded'] / dt:.3e}/s", flush=True)
    for comp in st["components"]:
        for a in comp["attempts"]:
            lay = a["layers"]
            print("  k", a["k"], a["outcome"], "rounds", len(lay), "expanded",
                  sum(l["expanded"] for l in lay), "max_layer", max([l["emitted"] for l in lay] or [0]),
                  "overflowed", a["overflowed"], flush=True)
