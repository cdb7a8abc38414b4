mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 2>&1 | tail -1
python - <<'PY'
import os, sys, json
sys.path.insert(0, os.getcwd()); sys.path.insert(0, "tests")
from paper_1709_09990_b200 import elimtw as E, generators as G
from checkers import RefLib
for name, rows in (("queen6_6", G.queen_graph(6, 6)), ("myciel4", G.myciel(4))):
    g = E.Graph.from_rows(rows)
    for mode in ("bloom", "exact"):
        o = E.Options(dedup=mode, use_mmw=True)
        E.solve(g, o)
        E.timer_begin(); r = E.solve(g, o); ms = E.timer_end()
        st = json.loads(r.stats_json)
        print(name, mode, "mmw", r.value, f"{ms:.1f} ms", st["totals"])
PY
