# Round-2 call AD: 32-byte (full-sector) records vs 16-byte; the part kernel without TMA as the common base.
O=gpurun_out/r02ad; mkdir -p $O
timeout 900 python tools/ab_lib.py tools/ab/libelimtw_notma.so tools/ab/libelimtw_rec32.so 3 > $O/ab_rec32.txt 2>&1; cat $O/ab_rec32.txt
for v in notma rec32; do
ETWG_LIB=$PWD/tools/ab/libelimtw_$v.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_exact -c 4000 --csv --log-file $O/launches_$v.csv python tools/prof_decide.py 22 exact > /dev/null 2>&1
python - $O/launches_$v.csv <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
per = {}
for r in rows[h + 1:]:
    d = dict(zip(rows[h], r))
    per.setdefault((d["ID"], d["Kernel Name"].split("(")[0]), {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
best = {}
for (i, k), m in per.items():
    if k not in best or m["gpu__time_duration.sum"] > best[k]["gpu__time_duration.sum"]:
        best[k] = m
for k, m in best.items():
    print(sys.argv[1], k, "longest launch ms %.2f read GB %.1f write GB %.1f" % (m["gpu__time_duration.sum"] / 1e6, m["dram__bytes_read.sum"] / 1e9, m["dram__bytes_write.sum"] / 1e9))
PY
done
