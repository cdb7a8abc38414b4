"""Per-config measurements (not the bench line): every BASELINE.json config on
one B200 beside the reference CPU solver (oracle/_ref) on the same box.
Writes profiles/<out>.json and prints a markdown table.
Test infrastructure (uses the reference build as the CPU arm).
Usage: python tests/measure_configs.py out_name [ref_threads]

  cfg1  myciel4, exact, default options (1 GPU vs reference 1 thread and all)
  cfg2  queen6_6, --mmw, Bloom
  cfg3  G(40,0.3) seed 1, default options (Bloom) and exact
  cfg4  G(48,0.2) seed 1, exact and Bloom, max_layer_states 2^31 (reference:
        too long — see bench.py's bounded sample)
  cfg5  8x8 grid + 6 chords (n=64) and 8x9 grid + 6 chords (n=72, 128-bit),
        default cap: the layers outgrow any cap, both report a lower bound
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))  # tests/ -> repo
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_1709_09990_b200 import elimtw as E, generators as G  # noqa: E402
from checkers import RefLib  # noqa: E402  (test infrastructure: the CPU reference)

out_name = sys.argv[1] if len(sys.argv) > 1 else "configs"
threads = int(sys.argv[2]) if len(sys.argv) > 2 else (os.cpu_count() or 1)
ref = RefLib()


def gpu(rows, reps=3, **kw):
    g = E.Graph.from_rows(rows)
    opts = E.Options(**kw)
    E.solve(g, opts)  # warm-up (allocations)
    best = None
    for _ in range(reps):
        E.timer_begin()
        r = E.solve(g, opts)
        ms = E.timer_end()
        best = ms if best is None else min(best, ms)
    st = json.loads(r.stats_json)
    return {"kind": r.kind, "value": r.value, "ms": best, "expanded": st["totals"]["expanded"]}


def cpu(rows, thr, **kw):
    t0 = time.perf_counter()
    r = ref.solve(rows, threads=thr, **kw)
    dt = time.perf_counter() - t0
    st = json.loads(r["stats"])
    return {"kind": r["kind"], "value": r["value"], "ms": 1e3 * dt, "expanded": st["totals"]["expanded"]}


rows_m4 = G.myciel(4)
rows_q6 = G.queen_graph(6, 6)
rows_40 = G.random_graph(1, 40, 0.3)
rows_48 = G.random_graph(1, 48, 0.2)
res = []


def add(cfg, name, g, c=None, c1=None):
    row = {"cfg": cfg, "case": name, "gpu": g}
    if c:
        row["ref_all_threads"] = c
    if c1:
        row["ref_1_thread"] = c1
    res.append(row)
    print(json.dumps(row), flush=True)


add(1, "myciel4 exact", gpu(rows_m4, dedup="exact"), cpu(rows_m4, threads, dedup="exact"),
    cpu(rows_m4, 1, dedup="exact"))
add(2, "queen6_6 mmw bloom", gpu(rows_q6, dedup="bloom", use_mmw=True),
    cpu(rows_q6, threads, dedup="bloom", mmw=True), cpu(rows_q6, 1, dedup="bloom", mmw=True))
add(3, "G(40,0.3) bloom (defaults)", gpu(rows_40, dedup="bloom"), cpu(rows_40, threads, dedup="bloom"))
add(3, "G(40,0.3) exact", gpu(rows_40, dedup="exact"), cpu(rows_40, threads, dedup="exact"))
add(4, "G(48,0.2) exact cap 2^31", gpu(rows_48, reps=2, dedup="exact", max_layer_states=1 << 31))
add(4, "G(48,0.2) bloom cap 2^31", gpu(rows_48, reps=1, dedup="bloom", max_layer_states=1 << 31))
for r_, c_ in ((8, 8), (8, 9)):
    rows = G.grid_with_chords(r_, c_, 6, 7)
    add(5, f"{r_}x{c_} grid + 6 chords (seed 7), exact, cap 10M", gpu(rows, reps=1, dedup="exact"),
        cpu(rows, threads, dedup="exact") if r_ * c_ <= 64 else None)

with open(os.path.join(ROOT, "profiles", f"{out_name}.json"), "w") as f:
    json.dump({"ref_threads": threads, "device": E.device_info()["name"], "rows": res}, f, indent=1)
print("\n| cfg | case | GPU result | GPU ms | expanded | GPU states/s | ref ms (all thr) | ref ms (1 thr) |")
print("|---|---|---|---|---|---|---|---|")
for row in res:
    g, c, c1 = row["gpu"], row.get("ref_all_threads"), row.get("ref_1_thread")
    print(f"| {row['cfg']} | {row['case']} | {g['kind']} {g['value']} | {g['ms']:.1f} | {g['expanded']} | "
          f"{g['expanded'] / (g['ms'] / 1e3):.3g} | {c['ms']:.0f} ({c['kind']} {c['value']})"
          if c else f"| {row['cfg']} | {row['case']} | {g['kind']} {g['value']} | {g['ms']:.1f} | "
          f"{g['expanded']} | {g['expanded'] / (g['ms'] / 1e3):.3g} | — ", end="")
    print(f" | {c1['ms']:.0f} |" if c1 else " | — |")
