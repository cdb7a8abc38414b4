mkdir -p gpurun_out
cat > /tmp/ab.py <<'PY'
import os, sys, time
sys.path.insert(0, os.getcwd())
from paper_1709_09990_b200 import elimtw as E, generators as G
rows = G.random_graph(1, 48, 0.2)
E.decide(rows, 22, dedup="exact", cap=1 << 31, keep_layers=False)
E.set_profiling(True); E.reset_times()
E.decide(rows, 22, dedup="exact", cap=1 << 31, keep_layers=False)
t = E.times(); print({k: round(t[k], 1) for k in ("expand_ms", "insert_ms", "append_ms")})
PY
python /tmp/ab.py
ETWG_DEBUG=32 python /tmp/ab.py
