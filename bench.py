#!/usr/bin/env python
"""Benchmark: wavefront states expanded per second (BASELINE.json metric).

Workload (BASELINE cfg 3, the config the metric is quoted at 1/2/4/8 GPUs):
G(n=40, p=0.3) seed 1 from the reference's own generator
(proj/tests/helpers.hpp:12-20), one *step* = one full etw_solve with the
reference defaults (Bloom dedup, biconnected split, clique, improvement
edges, start k = max(clique-1, MMW)), i.e. the full k sweep k=14..22 to the
exact treewidth 22. Unit of work = LayerStats::expanded (dp.cpp:77), summed.

  value  states expanded / device time of the K timed steps (CUDA events on
         the engine stream, one bracket per step; L2 flushed between steps)
  e2e    the same metric through the C ABI from host text: etw_graph_parse +
         etw_solve + etw_result_stats_json, wall clock per step, H2D/D2H
         bytes counted by the engine
  roofline  dominant kernel class from a profiled pass (per-launch CUDA
         events), algorithmic bytes per SURVEY §8d / DESIGN.md
  cpu_baseline  the reference (oracle/_ref) solving the same workload on the
         host cores (rank 0, N=1 only)

--impl reference runs the reference CPU solver (oracle/_ref, all host
threads) on the same workload and prints its line with "impl": "reference".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOAD = {"workload": "G(40,0.3) seed 1, full k sweep to exact treewidth (etw_solve)",
            "graph": "random_graph(seed=1, n=40, p=0.3)", "n": 40, "m": 251, "seed": 1,
            "dedup": "bloom", "split": "biconnected", "clique": True, "improvement": True,
            "start_k": "auto", "max_layer_states": 10_000_000, "emit_order": False,
            "l2": "flushed between steps (256 MiB write)", "parallelism": "dp1"}
METRIC = "wavefront states expanded/sec"
UNIT = "states/s"


def env_rank():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def workload_rows():
    from paper_1709_09990_b200 import generators as G
    return G.random_graph(1, 40, 0.3)


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
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def solve_once(E, graph, opts):
    res = E.solve(graph, opts)
    st = json.loads(res.stats_json)
    return res, st["totals"]["expanded"]


def run_gpu(args):
    import torch

    from paper_1709_09990_b200 import elimtw as E
    from paper_1709_09990_b200 import generators as G

    rank, world, local = env_rank()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
        os.environ["ETWG_DEVICE"] = str(local)
    else:
        dist = None
    info = E.device_info()
    if not info["available"]:
        raise SystemExit("bench: no CUDA device for libelimtw")

    rows = workload_rows()
    text = G.to_gr(rows)
    graph = E.Graph.parse(text)
    opts = E.Options(dedup="bloom")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{torch.cuda.current_device()}")

    for _ in range(args.warmup):
        res, expanded = solve_once(E, graph, opts)
    assert res.value == 22, f"wrong treewidth {res.value}"

    # ---- timed region: K steps, device time per step (events) ----------
    E.reset_times()
    step_ms = []
    total_expanded = 0
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(torch.cuda.current_device()) as clk:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            E.timer_begin()
            res, expanded = solve_once(E, graph, opts)
            step_ms.append(E.timer_end())
            total_expanded += expanded
            assert res.value == 22
    torch.cuda.synchronize()
    t = E.times()
    launches = int(t["kernel_launches"])
    dev_ms = sum(step_ms)
    if dist:
        tt = torch.tensor([dev_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dev_ms = float(tt.item())
        ee = torch.tensor([float(total_expanded)], device="cuda")
        dist.all_reduce(ee)
        total_expanded = int(ee.item())
    value = total_expanded / (dev_ms / 1e3)

    # ---- e2e: C ABI from host text, wall clock -------------------------
    E.reset_times()
    t0 = time.perf_counter()
    e2e_expanded = 0
    for _ in range(args.steps):
        g2 = E.Graph.parse(text)
        res2, ex2 = solve_once(E, g2, opts)
        e2e_expanded += ex2
    e2e_s = time.perf_counter() - t0
    t2 = E.times()
    e2e = {"value": e2e_expanded / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": int(t2["h2d_bytes"] / args.steps),
           "d2h_bytes_per_step": int(t2["d2h_bytes"] / args.steps),
           "ms_per_step": 1e3 * e2e_s / args.steps,
           "path": "etw_graph_parse(text) + etw_solve + etw_result_stats_json"}

    # ---- roofline: profiled pass, per-launch events ---------------------
    E.reset_times()
    E.set_profiling(True)
    solve_once(E, graph, opts)
    E.set_profiling(False)
    p = E.times()
    roof = roofline(p)

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
            "scaling": "weak" if world > 1 else "strong", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (reference generator, fixed seed)", "config": WORKLOAD,
            "expanded_per_step": total_expanded // max(1, args.steps) // max(1, world),
            "treewidth": res.value, "e2e": e2e, "roofline": roof, "gpu_launches": launches,
            "clocks": clk.summary(), "device": info["name"]}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(rows)
    if rank == 0:
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


def roofline(p):
    """Dominant kernel class by total profiled time; algorithmic bytes per
    DESIGN.md §4 (expand: 2x8B per parent; insert: 68 B per offered child;
    append: 12 B per parent read + 12 B per state written)."""
    peak, peak_src = peaks()
    classes = {
        # Bloom pass 1: candidates + dedup, D = 4h = 68 B per offered child
        # plus the parent read and the mask write (2 x 8 B per parent)
        "k_bloom_dedup": (p["insert_ms"], p["insert_launches"], p["dedup_bytes"] + 16.0 * p["expanded"]),
        "k_expand": (p["expand_ms"], p["expand_launches"], 16.0 * p["expanded"]),
        "k_append": (p["append_ms"], p["append_launches"], p["layer_bytes"]),
        "k_bloom_clear": (p["clear_ms"], p["clear_launches"], None),
    }
    name, (ms, n, bytes_) = max(((k, v) for k, v in classes.items() if v[2] is not None),
                                key=lambda kv: kv[1][0])
    avg_ms = ms / max(1, n)
    per_launch = bytes_ / max(1, n)
    achieved = per_launch / (avg_ms / 1e3) / 1e9 if avg_ms > 0 else 0.0
    total_ms = sum(v[0] for v in classes.values())
    round_bytes = p["layer_bytes"] + p["dedup_bytes"]
    return {"bound": "hbm", "kernel": name, "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": None, "peak_source": peak_src,
            "avg_launch_us": 1e3 * avg_ms, "launches": int(n),
            "algorithmic_bytes_per_launch": per_launch,
            "share_of_wavefront_time": ms / total_ms if total_ms else None,
            "wavefront_round_GBps": round_bytes / (total_ms / 1e3) / 1e9 if total_ms else None,
            "kernel_ms": {k: v[0] for k, v in classes.items()}}


def reference_solve(rows, threads):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from checkers import RefLib
    ref = RefLib()
    t0 = time.perf_counter()
    r = ref.solve(rows, dedup="bloom", threads=threads)
    dt = time.perf_counter() - t0
    expanded = json.loads(r["stats"])["totals"]["expanded"]
    assert r["value"] == 22
    return expanded, dt


def cpu_baseline(rows):
    threads = os.cpu_count() or 1
    try:
        expanded, dt = reference_solve(rows, threads)
    except Exception as e:  # reference build missing on this box
        return {"value": None, "unit": UNIT, "cores": threads, "kind": "reference",
                "sample": f"unavailable: {e}"}
    return {"value": expanded / dt, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"one full solve of the same workload ({expanded} expanded states, "
                      f"{dt:.2f} s) by the reference elimtw core (oracle/_ref) with "
                      f"thread_count={threads}"}


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    rows = workload_rows()
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        reference_solve(rows, threads)
    total, secs = 0, 0.0
    for _ in range(args.steps):
        e, dt = reference_solve(rows, threads)
        total += e
        secs += dt
    value = total / secs
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (reference generator, fixed seed)", "config": WORKLOAD,
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": "full solve per step, reference elimtw core (oracle/_ref), "
                                       f"thread_count={threads}"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
