"""Virtual-shard timings of the bench workload (not a benchmark): the
G(48,0.2) exact solve on the single-device engine and on G = 2, 4, 8
virtual shards of one GPU (every shard's kernels on the same device, so the
G-shard time is the sum of the shards' work; projected G-GPU time = that /
G + the per-round collective cost). Stats must equal the single-device run.
Usage: python tools/shard_times.py [G ...]"""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1709_09990_b200 import elimtw as E, generators as G  # noqa: E402

g = E.Graph.from_rows(G.random_graph(1, 48, 0.2))
o = E.Options(dedup="exact", max_layer_states=1 << 31)


def timed(reps=2):
    E.solve(g, o)
    ts = []
    for _ in range(reps):
        E.timer_begin()
        r = E.solve(g, o)
        ts.append(E.timer_end() / 1e3)
    return min(ts), r


t1, r1 = timed()
out = {"single_s": t1, "expanded": json.loads(r1.stats_json)["totals"]["expanded"], "shards": {}}
for gs in [int(x) for x in sys.argv[1:]] or [2, 4, 8]:
    E.set_virtual_shards(gs)
    E.reset_times()
    t, r = timed()
    tm = E.times()
    out["shards"][gs] = {"s": t, "per_state_vs_single": t / t1, "same_stats": r.stats_json == r1.stats_json,
                         "exchange_GB": tm["exchange_bytes"] / 3 / 1e9, "launches": tm["kernel_launches"] / 3}
    E.set_virtual_shards(1)
print(json.dumps(out, indent=1))
