# Round-2 call AP: sibling swap pre-dedup in the scatter's producer warps.
O=gpurun_out/r02ap; mkdir -p $O
L=paper_1709_09990_b200/libelimtw.so
timeout 900 python tools/ab_lib.py tools/ab/libelimtw_noswap.so $L 3 > $O/ab_swap.txt 2>&1; cat $O/ab_swap.txt
for v in noswap default; do
  lib=$PWD/tools/ab/libelimtw_$v.so; [ $v = default ] && lib=$PWD/$L
  ETWG_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_exact --csv --log-file $O/k22_$v.csv python tools/k1_only.py > /dev/null 2>&1
  python - $O/k22_$v.csv $v <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
per = {}
for r in rows[h + 1:]:
    d = dict(zip(rows[h], r))
    per.setdefault((int(d["ID"]), d["Kernel Name"].split("(")[0].split("::")[-1]), {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
best = {}
for (i, k), m in per.items():
    if k not in best or m["gpu__time_duration.sum"] > best[k]["gpu__time_duration.sum"]:
        best[k] = m
for k, m in best.items():
    print(sys.argv[2], k, "ms %.2f  DRAM read %.1f GB write %.1f GB" % (m["gpu__time_duration.sum"] / 1e6, m["dram__bytes_read.sum"] / 1e9, m["dram__bytes_write.sum"] / 1e9))
PY
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_big_configs.py -x -q -m gpu > $O/parity.txt 2>&1; tail -2 $O/parity.txt
