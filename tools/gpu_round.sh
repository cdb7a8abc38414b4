mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_shard.py -x -q --timeout 600 2>&1 | tail -3
python - <<'PY'
import os, sys, time
sys.path.insert(0, os.getcwd())
from paper_1709_09990_b200 import elimtw as E, generators as G
rows = G.random_graph(1, 40, 0.3)
g = E.Graph.from_rows(rows)
for vs in (1, 2, 8):
    E.set_virtual_shards(vs)
    E.solve(g, E.Options(dedup="exact"))
    E.timer_begin(); r = E.solve(g, E.Options(dedup="exact")); ms = E.timer_end()
    print("G40 exact vshards", vs, f"{ms:.1f} ms", r.value)
E.set_virtual_shards(1)
PY
for vs in 2 8; do timeout 600 python bench.py --virtual-shards $vs --steps 2 --warmup 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('vs$vs', d['value'], d['ms_per_step'], d.get('exchange_GB_per_step'), d.get('rerun_rounds'), d['gpu_launches'])"; done
