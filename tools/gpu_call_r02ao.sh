# Round-2 call AO: emission alone (no K1), K1 alone (no emission), a second returning atomic per record.
O=gpurun_out/r02ao; mkdir -p $O
for f in 262144; do
  ETWG_DEBUG=$f timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:k_exact_scatter --csv --log-file $O/d_$f.csv python tools/k1_only.py > $O/d_$f.out 2>&1
  python - $O/d_$f.csv $f <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
per = {}
for r in rows[h + 1:]:
    d = dict(zip(rows[h], r))
    if d["Kernel Name"].find(", 1>") < 0: continue   # bucket-round instantiation only
    per.setdefault(int(d["ID"]), {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
last = per[max(per)]
print(sys.argv[2], "last bucket-round scatter launch: ms %.2f  DRAM read %.1f write %.1f GB  inst %.2e" % (
    last["gpu__time_duration.sum"] / 1e6, last["dram__bytes_read.sum"] / 1e9, last["dram__bytes_write.sum"] / 1e9, last["smsp__inst_executed.sum"]))
PY
  tail -1 $O/d_$f.out
done
