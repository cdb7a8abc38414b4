# Round-2 call H: half-word slot K1 A/B (register slots incl. isolated members).
O=gpurun_out/r02h; mkdir -p $O
L=paper_1709_09990_b200/libelimtw.so
for v in half8 half6 half10 half8m4 half6m4; do
  timeout 600 python tools/ab_lib.py $L tools/ab/libelimtw_$v.so 3 > $O/ab_$v.txt 2>&1; head -3 $O/ab_$v.txt
done
