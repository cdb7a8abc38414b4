"""Profiling helper (run under gpurun): finds the longest launch of a kernel
in a command's launch list, then captures exactly that launch with
`ncu --set full`. Usage: python tools/ncu_top.py <kernel-regex> <out-name> -- <cmd...>"""
import csv, os, re, subprocess, sys

regex, name = sys.argv[1], sys.argv[2]
cmd = sys.argv[sys.argv.index("--") + 1:]
os.makedirs("gpurun_out", exist_ok=True)
lst = f"{name}_launches.csv" if "/" in name else f"gpurun_out/{name}_launches.csv"
subprocess.run(["ncu", "--metrics", "gpu__time_duration.sum", "--clock-control", "none", "-k",
                f"regex:{regex}", "--csv", "--log-file", lst, *cmd], check=True,
               stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
rows = list(csv.reader(open(lst)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]
times = []
for r in rows[hdr + 1:]:
    if len(r) == len(h):
        d = dict(zip(h, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            times.append(float(d["Metric Value"].replace(",", "")))
best = max(range(len(times)), key=lambda i: times[i])
print(f"{len(times)} launches of {regex}; longest #{best}: {times[best] / 1e3:.1f} us", flush=True)
subprocess.run(["ncu", "--set", "full", "--clock-control", "none", "--import-source", "on", "-k",
                f"regex:{regex}", "-s", str(best), "-c", "1", "-f", "-o", name if "/" in name else f"gpurun_out/{name}", *cmd],
               check=True, stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
print("captured", name)
