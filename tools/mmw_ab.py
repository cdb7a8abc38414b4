"""MMW timing probe (not a benchmark): solves with minor-min-width pruning in
fresh processes under two environments (default: ETWG_DEBUG=0 vs 256, i.e.
the default scatter vs forced warp-per-parent candidate evaluation) and
checks the stats JSON is identical.
Usage: python tools/mmw_ab.py [reps] [VAR=v,... VAR=v,...]"""
import json, os, subprocess, sys

CODE = r"""
import json, sys, time
sys.path.insert(0, '.')
from paper_1709_09990_b200 import elimtw as E, generators as G
out = {}
for name, rows in (("queen6_6", G.queen_graph(6, 6)), ("myciel4", G.myciel(4)),
                   ("g40", G.random_graph(1, 40, 0.3))):
    g = E.Graph.from_rows(rows)
    for dedup in ("exact", "bloom"):
        o = E.Options(dedup=dedup, use_mmw=True, max_layer_states=1 << 31)
        E.solve(g, o)
        ts = []
        for _ in range(int(sys.argv[1])):
            t0 = time.perf_counter(); r = E.solve(g, o); ts.append(time.perf_counter() - t0)
        out[name + "/" + dedup] = [min(ts), r.value, r.stats_json if dedup == "exact" else r.value]
print(json.dumps(out))
"""
reps = sys.argv[1] if len(sys.argv) > 1 else "3"
specs = sys.argv[2:4] if len(sys.argv) > 3 else ["ETWG_DEBUG=0", "ETWG_DEBUG=256"]
res = []
for spec in specs:
    env = dict(os.environ)
    for kv in filter(None, spec.split(",")):
        k, v = kv.split("=", 1)
        env[k] = v
    p = subprocess.run([sys.executable, "-c", CODE, reps], env=env, capture_output=True, text=True, timeout=1800)
    if p.returncode:
        print("failed", p.stderr[-2000:]); sys.exit(1)
    res.append(json.loads(p.stdout.strip().splitlines()[-1]))
for k in res[0]:
    a, b = res[0][k], res[1][k]
    print(f"{k:18s} tw {a[1]}  {specs[0]} {a[0]*1e3:9.1f} ms  {specs[1]} {b[0]*1e3:9.1f} ms  identical {a[2] == b[2]}")
