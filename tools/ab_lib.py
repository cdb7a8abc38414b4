"""A/B timing of two builds of libelimtw.so (not a benchmark): runs the
G(48,0.2) exact solve in a fresh process per library (ETWG_LIB) and checks
that the stats JSON is identical. Usage: python tools/ab_lib.py libA libB [reps] [exact|bloom]"""
import json, os, subprocess, sys

CODE = r"""
import json, sys, time
sys.path.insert(0, '.')
from paper_1709_09990_b200 import elimtw as E, generators as G
g = E.Graph.from_rows(G.random_graph(1, 48, 0.2))
o = E.Options(dedup=sys.argv[2], max_layer_states=1 << 31)
E.solve(g, o)
ts = []
for _ in range(int(sys.argv[1])):
    t0 = time.perf_counter(); r = E.solve(g, o); ts.append(time.perf_counter() - t0)
q = E.Graph.from_rows(G.queen_graph(6, 6))
t0 = time.perf_counter(); rq = E.solve(q, E.Options(dedup='bloom', use_mmw=True)); tq = time.perf_counter() - t0
h = E.Graph.from_rows(G.grid_with_chords(8, 9, 6, 7))
t0 = time.perf_counter(); rh = E.solve(h, E.Options(dedup='exact')); th = time.perf_counter() - t0
print(json.dumps({"g48": sorted(ts), "stats": r.stats_json, "queen": [tq, rq.stats_json], "n72": [th, rh.stats_json]}))
"""

reps = sys.argv[3] if len(sys.argv) > 3 else "3"
dedup = sys.argv[4] if len(sys.argv) > 4 else "exact"
outs = []
for spec in sys.argv[1:3]:
    # "path.so" or "path.so@VAR=value,VAR2=value" (extra environment for that run)
    lib, _, extra = spec.partition("@")
    env = dict(os.environ, ETWG_LIB=os.path.abspath(lib))
    for kv in filter(None, extra.split(",")):
        k, v = kv.split("=", 1)
        env[k] = v
    p = subprocess.run([sys.executable, "-c", CODE, reps, dedup], env=env, capture_output=True, text=True, timeout=900)
    if p.returncode:
        print(lib, "failed", p.stderr[-2000:]); sys.exit(1)
    outs.append(json.loads(p.stdout.strip().splitlines()[-1]))
for lib, o in zip(sys.argv[1:3], outs):
    print(f"{lib}: g48 {['%.3f' % t for t in o['g48']]}  queen6_6 mmw {o['queen'][0]:.3f}s  n72 {o['n72'][0]:.3f}s")
a, b = outs


def diff(x, y, path=""):
    if type(x) is not type(y):
        return [path]
    if isinstance(x, dict):
        return [d for k in sorted(set(x) | set(y)) for d in diff(x.get(k), y.get(k), f"{path}.{k}")]
    if isinstance(x, list):
        if len(x) != len(y):
            return [f"{path}[len {len(x)} vs {len(y)}]"]
        return [d for i, (u, v) in enumerate(zip(x, y)) for d in diff(u, v, f"{path}[{i}]")]
    return [] if x == y else [f"{path}: {x} vs {y}"]


print("stats identical:", a["stats"] == b["stats"], a["queen"][1] == b["queen"][1], a["n72"][1] == b["n72"][1])
for d in diff(json.loads(a["stats"]), json.loads(b["stats"]))[:12]:
    print("  g48 differs at", d)
