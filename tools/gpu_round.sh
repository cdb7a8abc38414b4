mkdir -p gpurun_out
cat > /tmp/vs.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
from paper_1709_09990_b200 import elimtw as E, generators as G
E.set_virtual_shards(2)
g = E.Graph.from_rows(G.random_graph(1, 48, 0.2))
o = E.Options(dedup="exact", max_layer_states=1 << 31)
for _ in range(2):
    E.solve(g, o)
PY
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_vs2e_g48.csv python /tmp/vs.py > /dev/null 2>&1
