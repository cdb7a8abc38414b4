"""Probe (not a benchmark): candidate exactly-solvable instances above 64
vertices for the 128-bit path (BASELINE cfg 5b). One subprocess per instance
with a time limit. Usage: python tools/probe_wide.py"""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r"""
import json, sys, time
sys.path.insert(0, %r)
from paper_1709_09990_b200 import elimtw as E, generators as G
spec = json.loads(sys.argv[1])
rows = eval(spec["expr"], {"G": G})
g = E.Graph.from_rows(rows)
t = time.perf_counter()
r = E.solve(g, E.Options(dedup="exact", max_layer_states=1 << 31, emit_order=True))
dt = time.perf_counter() - t
st = json.loads(r.stats_json)
w, ok = g.check_order(r.order) if r.kind == "exact" else (None, None)
print(json.dumps({"inst": spec["expr"], "n": g.vertex_count, "m": g.edge_count, "tw": r.value, "kind": r.kind,
                  "s": round(dt, 3), "expanded": st["totals"]["expanded"], "order_width": w, "valid": ok,
                  "attempts": [a["k"] for c in st["components"] for a in c["attempts"]]}))
""" % ROOT
insts = ["G.queen_graph(8, 9)", "G.random_graph(1, 72, 0.5)", "G.random_graph(1, 72, 0.6)",
         "G.random_graph(1, 72, 0.7)", "G.random_graph(2, 80, 0.6)", "G.random_graph(1, 96, 0.75)"]
for expr in insts:
    try:
        p = subprocess.run([sys.executable, "-c", CODE, json.dumps({"expr": expr})], capture_output=True,
                           text=True, timeout=int(os.environ.get("PROBE_TIMEOUT", "150")))
        print(p.stdout.strip() or p.stderr[-500:], flush=True)
    except subprocess.TimeoutExpired:
        print(json.dumps({"inst": expr, "timeout": True}), flush=True)
