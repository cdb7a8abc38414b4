# Round-2 call AW: swap window over adjacent tile pairs (64 parents), with / without a 64-register cap.
O=gpurun_out/r02aw; mkdir -p $O
L=paper_1709_09990_b200/libelimtw.so
timeout 900 python tools/ab_lib.py $L tools/ab/libelimtw_swappair.so 3 > $O/ab_pair.txt 2>&1; cat $O/ab_pair.txt
timeout 900 python tools/ab_lib.py $L tools/ab/libelimtw_swappairm4.so 3 > $O/ab_pairm4.txt 2>&1; cat $O/ab_pairm4.txt
