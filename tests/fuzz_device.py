"""Randomised device-vs-oracle parity sweep (test infrastructure, not
collected by pytest): random graphs, k, forbidden sets, caps, dedup and MMW
modes, 64- and 128-bit keys, single device and 2..8 virtual shards with
random replicated-prefix thresholds. Exact mode must match the oracle's
counters and state sets (and, on one device, its layer order and
histories); Bloom mode its verdict with subset layers.
Usage: python tests/fuzz_device.py [seconds] [seed]"""
import os
import random
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)
from checkers import Oracle  # noqa: E402
from paper_1709_09990_b200 import elimtw as E, generators as G  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300
rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
oracle = Oracle()
t0 = time.time()
cases = fails = 0
while time.time() - t0 < budget:
    wide = rng.random() < 0.2
    n = rng.randint(66, 100) if wide else rng.randint(5, 34)
    p = (rng.uniform(2.0, 6.0) / n) if wide else rng.uniform(0.1, 0.5)
    rows = G.random_graph(rng.randrange(1 << 30), n, p)
    k = rng.randint(max(1, n // 6), max(2, n // 2))
    forbidden = 0
    if rng.random() < 0.3:
        for v in rng.sample(range(n), rng.randint(1, min(4, n - 1))):
            forbidden |= 1 << v
    mmw = (not wide) and n <= 16 and rng.random() < 0.3
    cap = rng.choice([10_000_000, 10_000_000, rng.randint(5, 3000)])
    rounds = rng.randint(3, 7) if wide else -1
    shards = rng.choice([1, 1, 2, 3, 5, 8])
    handoff = rng.choice([0, 50, 1000])
    E.set_virtual_shards(shards)
    E.set_shard_handoff(handoff)
    for dedup in ("exact", "bloom"):
        cases += 1
        try:
            a = E.decide(rows, k, forbidden=forbidden, dedup=dedup, mmw=mmw, cap=cap, rounds=rounds)
            b = oracle.decide(rows, k, forbidden=forbidden, dedup=dedup, mmw=mmw, cap=cap, rounds=rounds)
            ok = a.outcome == b.outcome
            if dedup == "exact" and not b.overflowed:
                ok = ok and [x.tuple() for x in a.rounds] == [x.tuple() for x in b.rounds]
                ok = ok and [sorted(s for s, _ in l) for l in a.layers] == [sorted(s for s, _ in l) for l in b.layers]
                if shards == 1:
                    ok = ok and a.layers == b.layers and (a.witness_set, a.witness_hist) == (b.witness_set, b.witness_hist)
            elif dedup == "exact":  # truncated: counters agree up to the first overflow
                first = next(i for i, x in enumerate(b.rounds) if x.overflowed)
                ok = ok and [x.tuple() for x in a.rounds[:first + 1]] == [x.tuple() for x in b.rounds[:first + 1]]
            elif not b.overflowed:
                ex = oracle.decide(rows, k, forbidden=forbidden, dedup="exact", mmw=mmw, cap=cap, rounds=rounds)
                if a.layers and ex.layers:
                    ok = ok and set(s for s, _ in a.layers[0]) <= set(s for s, _ in ex.layers[0])
        except Exception as e:  # noqa: BLE001
            ok = False
            print("EXC", repr(e))
        if not ok:
            fails += 1
            print("FAIL", dict(n=n, p=round(p, 3), k=k, forbidden=hex(forbidden), mmw=mmw, cap=cap,
                               rounds=rounds, shards=shards, handoff=handoff, dedup=dedup), flush=True)
E.set_virtual_shards(1)
print(f"{cases} cases, {fails} failures in {time.time() - t0:.0f} s")
sys.exit(1 if fails else 0)
