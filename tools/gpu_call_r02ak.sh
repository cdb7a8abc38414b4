# Round-2 call AK: what bounds the emission (atomic return vs store), lane unroll 3/4, bench.
O=gpurun_out/r02ak; mkdir -p $O
for f in 0 16384 32768 65536; do
  ETWG_DEBUG=$f timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_exact_scatter --csv \
     --log-file $O/diag_$f.csv python tools/k1_only.py > $O/diag_$f.out 2>&1
  python - "$O/diag_$f.csv" <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
per = {}
for r in rows[h + 1:]:
    d = dict(zip(rows[h], r))
    per.setdefault(int(d["ID"]), {})[d["Metric Name"]] = (d["Metric Value"], d["Metric Unit"])
best = max(per.values(), key=lambda m: float(m["gpu__time_duration.sum"][0].replace(",", "")))
print(sys.argv[1], best)
PY
done
L=paper_1709_09990_b200/libelimtw.so
timeout 900 python tools/ab_lib.py $L tools/ab/libelimtw_lu3.so 3 > $O/ab_lu3.txt 2>&1; cat $O/ab_lu3.txt
timeout 900 python tools/ab_lib.py tools/ab/libelimtw_lu4.so tools/ab/libelimtw_lu3.so 3 > $O/ab_lu4.txt 2>&1; cat $O/ab_lu4.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; tail -c 400 $O/bench.json
