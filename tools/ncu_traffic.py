"""Summarises ncu --set full captures of the dominant kernels into
profiles/<out>.json: per launch DRAM traffic (dram__bytes_read.sum +
dram__bytes_write.sum), duration, and the launch's algorithmic bytes
 taken from the decide's largest round (the longest launch
ncu_top.py captured). Usage:
  python tools/ncu_traffic.py out.json decide_stats.txt kernel[/G]=rep ...
decide_stats.txt: the per-round lines of tools/prof_decide.py
(round expanded emitted duplicates)."""
import csv, json, subprocess, sys

out, stats_path = sys.argv[1], sys.argv[2]
rounds = []
for line in open(stats_path):
    p = line.split()
    if len(p) == 4 and all(x.isdigit() for x in p):
        rounds.append(tuple(int(x) for x in p))
r, E, U, D = max(rounds, key=lambda t: t[2] + t[3])
P = U + D
# child records actually written (after the scatter's sibling swap
# pre-dedup; ETWG_TRACE prints them per round): RECORDS=<n>, default P
REC = int(__import__("os").environ.get("RECORDS", P))
alg = {  # W = 1 (n <= 64) exact mode, bytes per launch
    "k_exact_scatter": 16 * E + 16 * REC,
    "k_exact_part": 16 * REC + 8 * U,
    "k_append": 20 * E + 12 * U,
    "k_route": 8 * E + 16 * P,
    "k_owner": 16 * P + 12 * U,
    # global-table rounds (default for one-word exact rounds): one 16-byte
    # slot read per offered child, one slot written per distinct key; the
    # mark pass streams the table (TAB_SLOTS slots, from the decide's trace)
    "k_exact_scatter@gtab": 16 * E + 16 * P + 16 * U,
    "k_tab_mark": 16 * int(__import__("os").environ.get("TAB_SLOTS", "0")) + 24 * U,
}


def metrics(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h, units, v = rows[0], rows[1], rows[2]
    d = dict(zip(h, v))
    u = dict(zip(h, units))

    def val(k):
        x = float(d[k].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                 "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}.get(u.get(k, ""), 1)
        return x * scale
    return {"dram_bytes": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
            "duration_s": val("gpu__time_duration.sum"),
            "ipc": val("sm__inst_executed.avg.per_cycle_active"),
            "issue_pct": val("sm__issue_active.avg.pct_of_peak_sustained_elapsed"),
            "sm_pct": val("sm__throughput.avg.pct_of_peak_sustained_elapsed")}


res = {"round": {"index": r, "expanded": E, "emitted": U, "offered": P, "records": REC}}
for arg in sys.argv[3:]:
    name, rep = arg.split("=", 1)
    shards = 1
    if "/" in name:  # kernel/G: one of G virtual shards' launches (1/G of the round)
        name, g = name.split("/")
        shards = int(g)
    m = metrics(rep)
    a = alg[name] / shards
    res[name] = {"traffic_bytes": m["dram_bytes"], "algorithmic_bytes": a,
                 "traffic_over_algorithmic": m["dram_bytes"] / a, "duration_ms": 1e3 * m["duration_s"],
                 "algorithmic_GBps": a / m["duration_s"] / 1e9, "dram_GBps": m["dram_bytes"] / m["duration_s"] / 1e9,
                 "ipc": m["ipc"], "issue_slots_busy_pct": m["issue_pct"], "sm_throughput_pct": m["sm_pct"]}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
