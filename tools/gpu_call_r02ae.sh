# Round-2 call AE: warp-specialised scatter with 1 / 2 / 4 producer warps per 8-warp CTA.
O=gpurun_out/r02ae; mkdir -p $O
L=paper_1709_09990_b200/libelimtw.so
timeout 900 python tools/ab_lib.py $L tools/ab/libelimtw_p2.so 3 > $O/ab_p2.txt 2>&1; cat $O/ab_p2.txt
timeout 900 python tools/ab_lib.py tools/ab/libelimtw_p1.so tools/ab/libelimtw_p2.so 3 > $O/ab_p1.txt 2>&1; cat $O/ab_p1.txt
