# Round-2 call K: warp pre-dedup A/B (records / atomics now bound the scatter).
O=gpurun_out/r02k; mkdir -p $O
L=paper_1709_09990_b200/libelimtw.so
for v in wdd wdd1k; do
  timeout 600 python tools/ab_lib.py $L tools/ab/libelimtw_$v.so 3 > $O/ab_$v.txt 2>&1; head -3 $O/ab_$v.txt
done
