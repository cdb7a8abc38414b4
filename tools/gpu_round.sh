mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_shard.py -q --timeout 900 > gpurun_out/shard_tests.txt 2>&1; tail -3 gpurun_out/shard_tests.txt
VSHARDS=2 ETWG_HANDOFF=0 timeout 300 python tools/prof_decide.py 22 exact 2 2>&1 | sed -n 2p
python - <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
from paper_1709_09990_b200 import elimtw as E, generators as G
g = E.Graph.from_rows(G.random_graph(1, 48, 0.2))
o = E.Options(dedup="exact", max_layer_states=1 << 31)
for vs in (2, 8):
    for mode in ("emitter", "owner"):
        E.set_virtual_shards(vs); E.set_shard_mode(mode)
        E.solve(g, o)
        E.timer_begin(); r = E.solve(g, o); ms = E.timer_end()
        print("vshards", vs, mode, r.value, f"{ms:.0f} ms")
PY
