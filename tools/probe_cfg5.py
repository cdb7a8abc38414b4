"""Probe (not a benchmark): BASELINE cfg 5 instances — 8x8 grid + chords
(n = 64, one-word masks) and 8x9 grid + chords (n = 72, the 128-bit path) —
full etw_solve in exact mode. Usage: python tools/probe_cfg5.py [chords] [seed]"""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1709_09990_b200 import elimtw as E, generators as G
chords = int(sys.argv[1]) if len(sys.argv) > 1 else 6
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 7
mmw = len(sys.argv) > 3 and sys.argv[3] == "mmw"
cap = int(sys.argv[4]) if len(sys.argv) > 4 else 1 << 31
insts = [("grid", 8, 8), ("grid", 8, 9)]
if os.environ.get("PROBE_RANDOM"):
    n, p_, s_ = os.environ["PROBE_RANDOM"].split(",")
    insts = [("random", int(n), (float(p_), int(s_)))]
for kind_, r, c in insts:
    if kind_ == "grid":
        g = E.Graph.from_rows(G.grid_with_chords(r, c, chords, seed))
    else:
        g = E.Graph.from_rows(G.random_graph(c[1], r, c[0]))
    t0 = time.perf_counter()
    res = E.solve(g, E.Options(dedup="exact", max_layer_states=cap, emit_order=True, use_mmw=mmw))
    dt = time.perf_counter() - t0
    st = json.loads(res.stats_json)
    width, valid = g.check_order(res.order) if res.kind == "exact" else (None, None)
    print(f"grid {r}x{c}+{chords} chords (seed {seed}) mmw={mmw} cap={cap}: n={g.vertex_count} m={g.edge_count} tw={res.value} "
          f"kind={res.kind} {dt:.2f}s expanded={st['totals']['expanded']} "
          f"({st['totals']['expanded'] / dt:.3e}/s) order width={width} valid={valid}", flush=True)
