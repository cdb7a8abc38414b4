mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 2>&1 | tail -1
timeout 300 python tools/prof_decide.py 22 exact 2 2>&1 | sed -n 2p
python - <<'PY'
import os, sys, json
sys.path.insert(0, os.getcwd())
from paper_1709_09990_b200 import elimtw as E, generators as G
for name, rows, kw in (("queen6_6 mmw bloom", G.queen_graph(6, 6), dict(dedup="bloom", use_mmw=True)),
                       ("myciel4 exact", G.myciel(4), dict(dedup="exact")),
                       ("G40 bloom", G.random_graph(1, 40, 0.3), dict(dedup="bloom")),
                       ("G40 exact", G.random_graph(1, 40, 0.3), dict(dedup="exact")),
                       ("G48 exact", G.random_graph(1, 48, 0.2), dict(dedup="exact", max_layer_states=1 << 31))):
    g = E.Graph.from_rows(rows)
    o = E.Options(**kw)
    E.solve(g, o)
    E.timer_begin(); r = E.solve(g, o); ms = E.timer_end()
    print(name, r.value, f"{ms:.1f} ms", json.loads(r.stats_json)["totals"])
PY
