"""Explains the Bloom-mode state losses on the bench graph (not a benchmark).
1. Solves G(48,0.2) seed 1 in Bloom mode with ETWG_DEBUG=2048, which logs the
   first distinct keys the filter rejected (key, h1, h2, m) per decide.
2. For the first logged key: rebuilds the round's inserted key set (the exact
   output of the same round: the inputs agree up to the first loss), computes
   every key's 17 probe positions (h1 + i*h2) mod m (bloom.cpp:86-97) with a
   vectorised Murmur3 x86_32 (bloom.cpp:27-64), and lists the keys covering
   the rejected key's positions.
Usage: python tools/bloom_fp_explain.py"""
import json, os, re, subprocess, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CODE = r"""
import sys, json
sys.path.insert(0, %r)
from paper_1709_09990_b200 import elimtw as E, generators as G
g = E.Graph.from_rows(G.random_graph(1, 48, 0.2))
E.reset_times()
r = E.solve(g, E.Options(dedup="bloom", max_layer_states=1 << 31))
t = E.times()
print(json.dumps({"tw": r.value, "probed": t["bloom_probed"], "fp": t["bloom_fp"], "stats": r.stats_json}))
""" % ROOT
env = dict(os.environ, ETWG_DEBUG="2048", ETWG_TRACE="1")
p = subprocess.run([sys.executable, "-c", CODE], capture_output=True, text=True, env=env, timeout=600)
res = json.loads(p.stdout.strip().splitlines()[-1])
print("bloom solve: tw", res["tw"], "distinct keys probed", int(res["probed"]), "rejected", int(res["fp"]))
rounds = [l for l in p.stderr.splitlines() if "rejected by the filter" in l]
print("\n".join(rounds))
fps = []
for l in p.stderr.splitlines():
    m = re.match(r"\[fp\] k=(\d+) key=([0-9a-f]+):([0-9a-f]+) h1=([0-9a-f]+) h2=([0-9a-f]+) m=(\d+)", l)
    if m:
        fps.append((int(m[1]), int(m[3], 16), int(m[4], 16), int(m[5], 16), int(m[6])))
print("logged:", len(fps))
for f in fps[:8]:
    print("  k=%d key=%012x h1=%08x h2=%08x m=%d" % f)
if not fps:
    sys.exit(0)

from paper_1709_09990_b200 import elimtw as E, generators as G  # noqa: E402
M32 = np.uint64(0xFFFFFFFF)


def murmur8(keys, seed):
    keys = keys.astype(np.uint64)
    h = np.full(keys.shape, seed, dtype=np.uint64)
    for part in (keys & M32, keys >> np.uint64(32)):
        k = (part * np.uint64(0xcc9e2d51)) & M32
        k = ((k << np.uint64(15)) | (k >> np.uint64(17))) & M32
        k = (k * np.uint64(0x1b873593)) & M32
        h ^= k
        h = ((h << np.uint64(13)) | (h >> np.uint64(19))) & M32
        h = (h * np.uint64(5) + np.uint64(0xe6546b64)) & M32
    h ^= np.uint64(8)
    h ^= h >> np.uint64(16)
    h = (h * np.uint64(0x85ebca6b)) & M32
    h ^= h >> np.uint64(13)
    h = (h * np.uint64(0xc2b2ae35)) & M32
    h ^= h >> np.uint64(16)
    return h


k, key, h1, h2, m = fps[0]
assert int(murmur8(np.array([key], dtype=np.uint64), 0x9747B28C)[0]) == h1
assert int(murmur8(np.array([key], dtype=np.uint64), 0x5EEDBA5E)[0]) == h2
rows = G.random_graph(1, 48, 0.2)
st = json.loads(res["stats"])
comp = max(st["components"], key=lambda c: len(c["vertices"]))
block = [v - 1 for v in comp["vertices"]]
sub = [sum(1 << j for j, u in enumerate(block) if rows[v] >> u & 1) for v in block]
clique = E.max_clique(sub)
free = len(sub) - bin(clique).count("1")
ex = E.decide(E.improve_graph(sub, k), k, forbidden=clique, dedup="exact", cap=1 << 31, keep_layers=False)
r = next(i for i, s in enumerate(ex.rounds) if (min(1 << 31, s.expanded * free) * 24 + 63) // 64 * 64 == m)
print("first loss: k=%d round=%d, %d keys inserted, m=%d bits" % (k, r, ex.rounds[r].emitted, m))
run = E.decide(E.improve_graph(sub, k), k, forbidden=clique, dedup="exact", cap=1 << 31, rounds=r + 1)
keys = np.array([s for s, _ in run.layers[r]], dtype=np.uint64)
assert key in set(keys.tolist()), "rejected key is not a distinct key of the round"
H1 = murmur8(keys, 0x9747B28C)
H2 = murmur8(keys, 0x5EEDBA5E)
mine = [(h1 + i * h2) % m for i in range(1, 18)]
cover = {}
for i in range(1, 18):
    pos = (H1 + np.uint64(i) * H2) % np.uint64(m)
    hit = np.nonzero(np.isin(pos, np.array(mine, dtype=np.uint64)))[0]
    for j in hit.tolist():
        if int(keys[j]) != key:
            cover.setdefault(int(keys[j]), set()).add(mine.index(int(pos[j])) + 1)
print("rejected key's probes: ", mine)
print("covering keys:", len(cover))
for ck, idx in sorted(cover.items(), key=lambda kv: -len(kv[1]))[:20]:
    j = int(np.nonzero(keys == np.uint64(ck))[0][0])
    print("  %012x h1=%08x h2=%08x covers probes %s" % (ck, int(H1[j]), int(H2[j]), sorted(idx)))
