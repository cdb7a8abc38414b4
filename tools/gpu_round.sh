mkdir -p gpurun_out
python - <<'PY'
import os, sys, json
sys.path.insert(0, os.getcwd())
from paper_1709_09990_b200 import elimtw as E, generators as G
g = E.Graph.from_rows(G.random_graph(1, 48, 0.2))
o = E.Options(dedup="exact", max_layer_states=1 << 31)
r = E.solve(g, o)
open("gpurun_out/g48_stats.json", "w").write(r.stats_json)
for vs, ho in ((8, 1 << 19), (8, 0), (2, 1 << 19)):
    E.set_virtual_shards(vs); E.set_shard_handoff(ho)
    E.solve(g, o)
    E.timer_begin(); r = E.solve(g, o); ms = E.timer_end()
    print("vshards", vs, "handoff", ho, f"{ms:.0f} ms")
E.set_virtual_shards(1)
PY
