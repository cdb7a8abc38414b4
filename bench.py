#!/usr/bin/env python
"""Benchmark: wavefront states expanded per second (BASELINE.json metric).

Workload (BASELINE cfg 4, the n >= 48 random-graph config the north_star's
1/2/4/8-GPU scaling target names): G(n=48, p=0.2) seed 1 from the
reference's own generator (proj/tests/helpers.hpp:12-20); one *step* = one
full etw_solve (biconnected split, clique, improvement edges, start k =
max(clique-1, MMW)) sweeping k = 11..24 to the exact treewidth 24 in exact
dedup mode, with max_layer_states = 2^31 so no layer is truncated (the
reference default 10M would overflow at k >= 17 and return a lower bound).
Unit of work = LayerStats::expanded (dp.cpp:77), summed over the solve:
2,316,224,115 states per step.

  value     states expanded / device time of the K timed steps (CUDA events
            on the engine stream around each step, max over ranks)
  e2e       the same metric through the C ABI from host text:
            etw_graph_parse + etw_solve + etw_result_stats_json, wall clock
            per step (max over ranks), H2D/D2H bytes counted by the engine
  roofline  dominant kernel class from a profiled pass (per-launch CUDA
            events), algorithmic bytes per DESIGN.md §4
  cpu_baseline  the reference elimtw core (oracle/_ref) on the box's host
            cores, rank 0 at N=1: a bounded sample of the same sweep — the
            reference's decide on the first attempts (k = 11, 12, ...) of the
            same block with the same improved graphs and forbidden clique
  bloom     Bloom-mode false-positive probe, the bench graph in Bloom mode,
            and a Bloom-vs-exact timing on G(40,0.3) (BASELINE cfg 3), N=1 only

N > 1 (torchrun): every rank becomes one owner shard (paper_1709_09990_b200/
distributed.py; states routed to hash owners over NCCL each round) and all
ranks run the same solve; the total work per step is fixed (strong scaling).

--impl reference runs the reference CPU decide sample (oracle/_ref, all host
threads) and prints its line with "impl": "reference" (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_VERT, P_EDGE, SEED, TW = 48, 0.2, 1, 24
CAP = 1 << 31
WORKLOAD = {"workload": "G(48,0.2) seed 1, full k sweep 11..24 to exact treewidth 24 (etw_solve)",
            "graph": "random_graph(seed=1, n=48, p=0.2)", "n": N_VERT, "m": 241, "seed": SEED,
            "dedup": "exact", "split": "biconnected", "clique": True, "improvement": True,
            "start_k": "auto", "max_layer_states": CAP, "emit_order": False,
            "expanded_per_step": 2316224115,
            "l2": "flushed between steps (256 MiB write); layers up to 164M states exceed L2"}
METRIC = "wavefront states expanded/sec"
UNIT = "states/s"


def env_rank():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def workload_rows():
    from paper_1709_09990_b200 import generators as G
    return G.random_graph(SEED, N_VERT, P_EDGE)


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.samples = []
        if self.proc is None:
            return
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        for line in out.splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.samples.append(parts)

    def summary(self):
        if not getattr(self, "samples", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"],
                    "samples": 0}
        sm = [float(p[1]) for p in self.samples if p[1].replace(".", "").isdigit()]
        mx = [float(p[2]) for p in self.samples if p[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for p in self.samples for i in range(4)
                          if p[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def solve_once(E, graph, opts):
    res = E.solve(graph, opts)
    st = json.loads(res.stats_json)
    return res, st["totals"]["expanded"], st


def run_gpu(args):
    rank, world, local = env_rank()
    os.environ.setdefault("ETWG_DEVICE", str(local))
    import torch

    torch.cuda.set_device(local)
    from paper_1709_09990_b200 import distributed as D
    from paper_1709_09990_b200 import elimtw as E
    from paper_1709_09990_b200 import generators as G

    info = E.device_info()
    if not info["available"]:
        raise SystemExit("bench: no CUDA device for libelimtw")
    if world > 1:
        shard = D.init_shards(local)
    else:
        if args.virtual_shards > 1:  # diagnostics: the sharded path on one GPU
            E.set_virtual_shards(args.virtual_shards)
        shard = E.shard_info()

    rows = workload_rows()
    text = G.to_gr(rows)
    graph = E.Graph.parse(text)
    opts = E.Options(dedup="exact", max_layer_states=CAP)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")

    for _ in range(args.warmup):
        res, expanded, stats = solve_once(E, graph, opts)
    assert res.value == TW, f"wrong treewidth {res.value}"

    # ---- timed region: K steps, device time per step (events) ----------
    E.reset_times()
    step_ms = []
    total_expanded = 0
    D.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            D.barrier()
            E.timer_begin()
            res, expanded, stats = solve_once(E, graph, opts)
            step_ms.append(E.timer_end())
            total_expanded += expanded  # global counters: every rank sees the whole solve
            assert res.value == TW
    torch.cuda.synchronize()
    t = E.times()
    launches = int(t["kernel_launches"])
    dev_ms = D.max_over_ranks(sum(step_ms))
    value = total_expanded / (dev_ms / 1e3)

    # ---- e2e: C ABI from host text, wall clock -------------------------
    E.reset_times()
    D.barrier()
    t0 = time.perf_counter()
    e2e_expanded = 0
    for _ in range(args.steps):
        g2 = E.Graph.parse(text)
        res2, ex2, _ = solve_once(E, g2, opts)
        e2e_expanded += ex2
    e2e_s = D.max_over_ranks(time.perf_counter() - t0)
    t2 = E.times()
    e2e = {"value": e2e_expanded / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": int(t2["h2d_bytes"] / args.steps),
           "d2h_bytes_per_step": int(t2["d2h_bytes"] / args.steps),
           "ms_per_step": 1e3 * e2e_s / args.steps,
           "path": "etw_graph_parse(text) + etw_solve + etw_result_stats_json"}

    # ---- roofline ------------------------------------------------------
    if not shard["virtual"] and world == 1:
        E.reset_times()
        E.set_profiling(True)
        solve_once(E, graph, opts)
        E.set_profiling(False)
        roof = roofline(E.times())
    else:
        roof = sharded_roofline(t, dev_ms, shard["world"])

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (reference generator, fixed seed)",
            "config": dict(WORKLOAD, parallelism=f"owner-sharded x{world}" if world > 1 else "1 GPU"),
            "expanded_per_step": total_expanded // max(1, args.steps),
            "treewidth": res.value, "e2e": e2e, "roofline": roof, "gpu_launches": launches,
            "clocks": clk.summary(), "device": info["name"], "shards": shard}
    line["parity"] = golden_parity(stats)
    if shard["world"] > 1:
        line["exchange_GB_per_step"] = t["exchange_bytes"] / args.steps / 1e9
        line["rerun_rounds"] = int(t["reruns"])
    if rank == 0 and world == 1 and not args.no_extras and not shard["virtual"]:
        line["bloom"] = bloom_probe(E, G)
        line["cpu_baseline"] = cpu_baseline(rows, stats, budget_s=args.cpu_budget)
    if rank == 0:
        print(json.dumps(line), flush=True)


def golden_parity(stats):
    """The timed solve's stats against the reference's full sweep of the same
    workload (tests/golden/g48_ref.json, generated from the unmodified
    reference by tests/golden/make_big_goldens.py): every attempt's outcome,
    improvement edges and per-round counters, and the treewidth."""
    import hashlib
    path = os.path.join(ROOT, "tests", "golden", "g48_ref.json")
    if not os.path.exists(path):
        return {"golden": None, "match": None}
    raw = open(path, "rb").read()
    g = json.loads(raw)
    comp = max(stats["components"], key=lambda c: len(c["vertices"]))
    att = comp["attempts"]
    match = (stats["result"]["value"] == g["tw"] and len(att) == len(g["attempts"]) and all(
        (a["k"], a["outcome"], a["added_edges"]) == (w["k"], w["outcome"], w["added_edges"]) and
        [[l["round"], l["expanded"], l["emitted"], l["duplicates"], l["mmw_pruned"], l["overflowed"]]
         for l in a["layers"]] == w["layers"] for a, w in zip(att, g["attempts"])))
    ref_s = sum(a.get("ref_s", 0.0) for a in g["attempts"])
    return {"golden": "tests/golden/g48_ref.json", "golden_sha256": hashlib.sha256(raw).hexdigest()[:16],
            "rounds_compared": sum(len(w["layers"]) for w in g["attempts"]), "match": bool(match),
            # time to exact treewidth of the reference itself, recorded when the
            # golden was generated (not timed by this run): its decide on every
            # attempt of the same sweep
            "reference_time_to_tw_s": round(ref_s, 1),
            "reference_time_to_tw_hosts": "k=11..21 on 8 threads (dev container), k=22..24 on 14 threads "
                                          "of the GPU box's 16-core host (tests/golden/make_big_goldens.py)"}


def roofline(p):
    """Dominant kernel class by profiled device time; algorithmic bytes per
    launch from DESIGN.md §4 (engine-accounted per round)."""
    peak, peak_src = peaks()
    classes = {
        "k_exact_scatter": (p["expand_ms"], p["expand_launches"], p["expand_bytes"]),
        "k_exact_part": (p["insert_ms"], p["insert_launches"], p["insert_bytes"]),
        "k_append": (p["append_ms"], p["append_launches"], p["append_bytes"]),
    }
    name, (ms, n, bytes_) = max(classes.items(), key=lambda kv: kv[1][0])
    avg_ms = ms / max(1, n)
    per_launch = bytes_ / max(1, n)
    achieved = bytes_ / (ms / 1e3) / 1e9 if ms > 0 else 0.0
    total_ms = sum(v[0] for v in classes.values())
    round_bytes = sum(v[2] for v in classes.values())
    # DRAM traffic from the committed ncu --set full capture of this kernel's
    # longest launch (tools/ncu_traffic.py), scaled to the average launch
    traffic, traffic_src, alu = None, None, None
    tpath = os.path.join(ROOT, "profiles", "r02_traffic.json")
    if not os.path.exists(tpath):
        tpath = os.path.join(ROOT, "profiles", "r01_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tr = json.load(f).get(name)
        if tr:
            traffic = tr["traffic_over_algorithmic"] * per_launch
            traffic_src = (f"{os.path.relpath(tpath, ROOT)}: ncu --set full of the longest launch, DRAM bytes = "
                           f"{tr['traffic_over_algorithmic']:.2f} x algorithmic bytes, scaled to the average launch")
            if "issue_slots_busy_pct" in tr:
                alu = {"bound": "integer ALU issue", "issue_slots_busy_pct": tr["issue_slots_busy_pct"],
                       "ipc": tr["ipc"], "sm_throughput_pct": tr["sm_throughput_pct"],
                       "source": "same capture"}
    return {"bound": "hbm", "kernel": name, "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
            "compute_view": alu, "peak_source": peak_src,
            "avg_launch_us": 1e3 * avg_ms, "launches": int(n),
            "algorithmic_bytes_per_launch": per_launch,
            "share_of_wavefront_time": ms / total_ms if total_ms else None,
            "wavefront_round_GBps": round_bytes / (total_ms / 1e3) / 1e9 if total_ms else None,
            "kernel_ms": {k: v[0] for k, v in classes.items()},
            "kernel_GBps": {k: (v[2] / (v[0] / 1e3) / 1e9 if v[0] else None) for k, v in classes.items()},
            "children_offered": int(p["offered"]), "distinct_children": int(p["unique"]),
            "child_records": int(p.get("records", 0)),
            "algorithmic_bytes_note": "16 B per parent read + 16 B per winner-mask clear + 16 B per child "
                                      "record written (children left after the sibling swap pre-dedup)"}


def sharded_roofline(t, dev_ms, world):
    """N > 1: the whole sharded round (route + exchange + owner) against the
    aggregate HBM of the shards; exchange bytes reported against NVLink."""
    peak, peak_src = peaks()
    # per shard: one record (24 B) out and in per routed child, layer traffic
    bytes_ = t["layer_bytes"] + t["dedup_bytes"]
    achieved = bytes_ / (dev_ms / 1e3) / 1e9 / world
    return {"bound": "hbm", "kernel": "sharded round (k_route + exchange + k_owner)",
            "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": None, "peak_source": peak_src, "per": "GPU",
            "nvlink_GBps_per_gpu": t["exchange_bytes"] / world / (dev_ms / 1e3) / 1e9,
            "nvlink_peak_GBps": 900.0,
            "nvlink_peak_source": "NVLink 5, 900 GB/s per direction per GPU (SURVEY §8d)"}


def bloom_probe(E, G):
    """BASELINE cfg 3/4 'Bloom vs exact': (a) false positives measured on one
    round — the same input layer through expand_layer in exact and Bloom mode
    (Bloom novel keys are a subset of the exact ones; the difference are
    false positives) against the expected (1-e^{-hn/m})^h; (b) G(40,0.3)
    full solves in both modes."""
    out = {}
    try:
        rows = G.random_graph(1, 40, 0.3)
        run = E.decide(rows, 22, dedup="exact")
        big = max(range(len(run.layers)), key=lambda i: len(run.layers[i]))
        layer = run.layers[big]
        ex = E.expand_layer(rows, 22, layer, dedup="exact")
        bl = E.expand_layer(rows, 22, layer, dedup="bloom")
        u, b = ex.rounds[0].emitted, bl.rounds[0].emitted
        cap = min(10_000_000, max(1, len(layer) * 40))
        m = max(64, (cap * 24 + 63) // 64 * 64)
        expected = (1.0 - math.exp(-17.0 * u / m)) ** 17
        out["fp_probe"] = {"graph": "G(40,0.3) seed 1, k=22", "round_input_states": len(layer),
                           "exact_novel": u, "bloom_novel": b, "false_positives": u - b,
                           "measured_fp_rate": (u - b) / max(1, u), "expected_fp_rate": expected,
                           "filter_bits": m}
        g48 = E.Graph.from_rows(workload_rows())  # BASELINE cfg 4: Bloom vs exact on the bench graph
        opts = E.Options(dedup="bloom", max_layer_states=CAP)
        E.solve(g48, opts)
        E.reset_times()
        E.timer_begin()
        r = E.solve(g48, opts)
        ms = E.timer_end()
        tm = E.times()
        ex_n = json.loads(r.stats_json)["totals"]["expanded"]
        out["g48_bloom"] = {"treewidth": r.value, "expanded": ex_n, "ms": ms,
                            "states_per_s": ex_n / (ms / 1e3),
                            "distinct_keys_probed": int(tm.get("bloom_probed", 0)),
                            "rejected_by_filter": int(tm.get("bloom_fp", 0)),
                            "measured_fp_rate": tm.get("bloom_fp", 0) / max(1.0, tm.get("bloom_probed", 0)),
                            "fp_explained": "every rejected key shares its Murmur3 (h1, h2) pair -- all 17 "
                                            "probe positions -- with another distinct key of the same round "
                                            "(DESIGN.md 5.3, profiles/r02_bloom_fp_explained.txt)",
                            "path": "partitioned (filter > 2^28 bits): exact bucket dedup, then the "
                                    "reference's 17-probe filter per distinct child"}
        g40 = E.Graph.from_rows(rows)
        for mode in ("exact", "bloom"):
            E.solve(g40, E.Options(dedup=mode))
            E.timer_begin()
            r = E.solve(g40, E.Options(dedup=mode))
            ms = E.timer_end()
            ex_n = json.loads(r.stats_json)["totals"]["expanded"]
            out[f"g40_{mode}"] = {"treewidth": r.value, "expanded": ex_n, "ms": ms,
                                  "states_per_s": ex_n / (ms / 1e3)}
    except Exception as e:  # reported, never fatal
        out["error"] = repr(e)
    return out


# ---------------------------------------------------------------------------
# the reference's CPU implementation (oracle/_ref): bounded sample of the sweep

def _induced(rows, verts):
    idx = {v: i for i, v in enumerate(verts)}
    out = []
    for v in verts:
        r = 0
        x = rows[v]
        while x:
            low = x & -x
            u = low.bit_length() - 1
            if u in idx:
                r |= 1 << idx[u]
            x ^= low
        out.append(r)
    return out


def reference_sample(rows, threads, budget_s):
    """The reference's decide (dp.cpp:167-194, all host threads) on the
    attempts solve() makes first on the workload's largest biconnected block
    (solver.cpp:21-67: same block, forbidden clique, improved graph per k,
    exact dedup, the same layer cap), k = start, start+1, ... until
    `budget_s` of CPU time is spent. Returns (expanded, seconds, per-k)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from checkers import RefLib
    ref = RefLib()
    blocks = ref.split(rows, 2)
    verts = max(blocks, key=lambda b: len(b[0]))[0]
    sub = _induced(rows, verts)
    clique = ref.max_clique(sub)
    k = max(bin(clique).count("1") - 1, ref.mmw_lower_bound(sub))
    expanded, secs, per_k = 0, 0.0, []
    while secs < budget_s and k < len(sub):
        gk = ref.improve_graph(sub, k)
        t0 = time.perf_counter()
        run = ref.decide(gk, k, forbidden=clique, dedup="exact", cap=CAP, threads=threads,
                         keep_layers=False)
        dt = time.perf_counter() - t0
        e = sum(x.expanded for x in run.rounds)
        expanded += e
        secs += dt
        per_k.append((k, e, dt))
        if run.outcome == "feasible":
            break
        k += 1
    return expanded, secs, per_k


def cpu_baseline(rows, stats, budget_s):
    threads = os.cpu_count() or 1
    try:
        expanded, secs, per_k = reference_sample(rows, threads, budget_s)
    except Exception as e:  # reference build missing on this box
        return {"value": None, "unit": UNIT, "cores": threads, "kind": "reference",
                "sample": f"unavailable: {e!r}"}
    gpu = {a["k"]: sum(l["expanded"] for l in a["layers"])
           for c in stats["components"] for a in c["attempts"]}
    match = all(gpu.get(k) == e for k, e, _ in per_k)
    return {"value": expanded / secs, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": (f"reference decide (oracle/_ref, thread_count={threads}) on the first "
                       f"{len(per_k)} attempts k={per_k[0][0]}..{per_k[-1][0]} of the same sweep "
                       f"(largest block, improved graph, forbidden clique, exact dedup): "
                       f"{expanded} expanded states in {secs:.1f} s"),
            "per_k": [{"k": k, "expanded": e, "s": round(dt, 3)} for k, e, dt in per_k],
            "expanded_matches_gpu_attempts": match}


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    rows = workload_rows()
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        reference_sample(rows, threads, args.ref_budget)
    total, secs, desc = 0, 0.0, None
    for _ in range(args.steps):
        e, dt, per_k = reference_sample(rows, threads, args.ref_budget)
        total += e
        secs += dt
        desc = per_k
    value = total / secs
    sample = (f"per step: reference decide (oracle/_ref, thread_count={threads}) on the first "
              f"{len(desc)} attempts k={desc[0][0]}..{desc[-1][0]} of the workload's sweep "
              f"(largest block, improved graph, forbidden clique, exact dedup), "
              f"{total // args.steps} expanded states")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (reference generator, fixed seed)",
            "config": dict(WORKLOAD, parallelism="host threads"), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def torchrun_argv(argv, gpus, port=None):
    """The command that re-launches this bench as `gpus` ranks (one process
    per GPU, torchrun, rendezvous on 127.0.0.1)."""
    port = port or int(os.environ.get("MASTER_PORT", "29533"))
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]


def launch_ranks(args, argv):
    """`bench.py --gpus N` outside torchrun: N > 1 needs N ranks, so re-exec
    under torchrun; with fewer than N visible GPUs fail loudly instead of
    reporting a 1-GPU number as N."""
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(json.dumps({"metric": METRIC, "n_gpus": args.gpus, "error":
                          f"--gpus {args.gpus} needs {args.gpus} visible CUDA devices, found {have}"}),
              flush=True)
        raise SystemExit(2)
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # communicator init lines (ranks) on stderr
    raise SystemExit(subprocess.call(torchrun_argv(argv, args.gpus), env=env))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-extras", action="store_true", help="skip cpu_baseline and the Bloom probe")
    ap.add_argument("--virtual-shards", type=int, default=1,
                    help="diagnostics: run the owner-sharded path as G shards on one GPU")
    ap.add_argument("--cpu-budget", type=float, default=15.0, help="seconds of reference CPU work")
    ap.add_argument("--ref-budget", type=float, default=4.0,
                    help="seconds of reference CPU work per --impl reference step")
    args = ap.parse_args()
    _, world, _ = env_rank()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        launch_ranks(args, sys.argv[1:])
    if world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world} ranks were launched")
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
