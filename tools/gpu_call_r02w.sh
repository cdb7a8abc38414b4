# Round-2 call W: K1 / emission split under warp specialisation.
O=gpurun_out/r02w; mkdir -p $O
for f in 0 16384; do
  ETWG_DEBUG=$f timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_write.sum --clock-control none -k regex:k_exact_scatter --csv \
     --log-file $O/k1_$f.csv python tools/k1_only.py > $O/k1_$f.out 2>&1
  python - "$O/k1_$f.csv" <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
last = {}
for r in rows[h + 1:]:
    d = dict(zip(rows[h], r))
    last[d["Metric Name"]] = (d["ID"], d["Metric Value"], d["Metric Unit"])
print(sys.argv[1], last)
PY
done
