# Round-2 call AF: ncu --set full of the largest k_exact_scatter / k_exact_part_tma / k_append launch (k=22 decide), current build.
O=gpurun_out/r02af; mkdir -p $O
timeout 600 python tools/prof_decide.py 22 exact > $O/decide22.txt 2>&1; head -3 $O/decide22.txt
for k in k_exact_scatter k_exact_part_tma k_append; do
  timeout 900 python tools/ncu_top.py $k $O/$k -- python tools/prof_decide.py 22 exact > $O/ncu_$k.txt 2>&1; tail -1 $O/ncu_$k.txt
  ncu -i $O/$k.ncu-rep --page raw --csv > $O/$k.raw.csv 2>/dev/null
  ncu -i $O/$k.ncu-rep --page details --csv > $O/$k.details.csv 2>/dev/null
done
