# Round-2 call Q: slot-guard and one-multiply bucket hash A/B.
O=gpurun_out/r02q; mkdir -p $O
L=paper_1709_09990_b200/libelimtw.so
for v in guard mulhash; do
  timeout 400 python tools/ab_lib.py $L tools/ab/libelimtw_$v.so 3 > $O/ab_$v.txt 2>&1; head -3 $O/ab_$v.txt
done
