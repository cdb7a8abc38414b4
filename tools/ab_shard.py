"""A/B of two builds on G virtual shards (not a benchmark): the G(48,0.2)
exact solve per library in a fresh process; stats must match the
single-device solve. Usage: python tools/ab_shard.py libA libB [G] [mode]"""
import json, os, subprocess, sys

CODE = r"""
import json, sys, time
sys.path.insert(0, '.')
from paper_1709_09990_b200 import elimtw as E, generators as G
g = E.Graph.from_rows(G.random_graph(1, 48, 0.2))
o = E.Options(dedup='exact', max_layer_states=1 << 31)
single = E.solve(g, o).stats_json
E.set_virtual_shards(int(sys.argv[1]))
E.set_shard_mode(sys.argv[2])
E.solve(g, o)
ts = []
for _ in range(2):
    t0 = time.perf_counter(); r = E.solve(g, o); ts.append(time.perf_counter() - t0)
print(json.dumps({"t": sorted(ts), "same": r.stats_json == single}))
"""
shards = sys.argv[3] if len(sys.argv) > 3 else "2"
mode = sys.argv[4] if len(sys.argv) > 4 else "emitter"
for lib in sys.argv[1:3]:
    env = dict(os.environ, ETWG_LIB=os.path.abspath(lib))
    p = subprocess.run([sys.executable, "-c", CODE, shards, mode], env=env, capture_output=True, text=True, timeout=900)
    if p.returncode:
        print(lib, "failed", p.stderr[-2000:]); continue
    o = json.loads(p.stdout.strip().splitlines()[-1])
    print(f"{lib}: {shards} virtual shards ({mode}) {['%.3f' % t for t in o['t']]} stats==single: {o['same']}")
