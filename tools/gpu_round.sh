mkdir -p gpurun_out
cat > /tmp/w2.py <<'PY'
import os, sys, json
sys.path.insert(0, os.getcwd())
from paper_1709_09990_b200 import elimtw as E, generators as G
g = E.Graph.from_rows(G.grid_with_chords(8, 9, 6, 7))
o = E.Options(dedup="exact")
E.solve(g, o)
E.timer_begin(); r = E.solve(g, o); ms = E.timer_end()
print(r.kind, r.value, f"{ms:.1f} ms", json.loads(r.stats_json)["totals"]["expanded"])
PY
python /tmp/w2.py
ETWG_LIB=paper_1709_09990_b200/libelimtw_w2c.so python /tmp/w2.py
