# Round-2 call AL: mbarrier try_wait suspend-time hint in the warp-specialised scatter.
O=gpurun_out/r02al; mkdir -p $O
L=paper_1709_09990_b200/libelimtw.so
timeout 900 python tools/ab_lib.py tools/ab/libelimtw_nosusp.so $L 3 > $O/ab_susp.txt 2>&1; cat $O/ab_susp.txt
timeout 900 python tools/ab_lib.py tools/ab/libelimtw_susp1k.so $L 3 > $O/ab_susp1k.txt 2>&1; cat $O/ab_susp1k.txt
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:k_exact_scatter --csv --log-file $O/k22.csv python tools/k1_only.py > /dev/null 2>&1
python - $O/k22.csv <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
per = {}
for r in rows[h + 1:]:
    d = dict(zip(rows[h], r))
    per.setdefault(int(d["ID"]), {})[d["Metric Name"]] = d["Metric Value"]
print(max(per.values(), key=lambda m: float(m["gpu__time_duration.sum"].replace(",", ""))))
PY
