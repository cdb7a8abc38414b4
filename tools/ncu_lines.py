"""Per-CUDA-line stall samples of an ncu report (ncu --page source
--print-source=cuda,sass). Usage: python tools/ncu_lines.py rep [top]"""
import csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = None; lines = []; total = 0.0
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]; continue
    if len(r) > 8 and r[0].isdigit() and r[2] == "-":
        v = float(r[4] or 0); ins = float(r[7] or 0)
        lines.append((v, ins, f"{cur}:{r[0]}", r[1])); total += v
for v, ins, loc, s in sorted(lines, reverse=True)[:top]:
    print(f"{100 * v / max(total, 1):5.1f}%  inst={ins:12.0f}  {loc:22s} {s.strip()[:90]}")
