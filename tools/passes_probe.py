"""f4 rehearsal on the bench workload (not a benchmark): the G(48,0.2) solve
with every exact round split into P hash-range passes (ETWG_PASSES=P, the
out-of-HBM mechanism), in a fresh process per P; prints the time, the peak
record-buffer need per pass and whether the stats JSON equals the one-pass
solve. Usage: python tools/passes_probe.py P [P ...]"""
import json, os, subprocess, sys
CODE = r"""
import json, sys, time
sys.path.insert(0, '.')
from paper_1709_09990_b200 import elimtw as E, generators as G
g = E.Graph.from_rows(G.random_graph(1, 48, 0.2))
o = E.Options(dedup='exact', max_layer_states=1 << 31)
E.solve(g, o)
E.timer_begin(); r = E.solve(g, o); ms = E.timer_end()
print(json.dumps({"ms": ms, "stats": r.stats_json}))
"""
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
res = {}
for p in ["1"] + sys.argv[1:]:
    env = dict(os.environ, ETWG_PASSES=p)
    out = subprocess.run([sys.executable, "-c", CODE], env=env, cwd=root, capture_output=True, text=True, timeout=900)
    if out.returncode:
        print(p, "failed", out.stderr[-1000:]); continue
    res[p] = json.loads(out.stdout.strip().splitlines()[-1])
base = res.get("1")
for p, r in res.items():
    print(json.dumps({"passes": int(p), "ms": round(r["ms"], 1), "stats_equal_one_pass": base is not None and r["stats"] == base["stats"]}))
