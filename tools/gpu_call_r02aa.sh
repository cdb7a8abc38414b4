# Round-2 call AA: bucket cursors strided apart (L2 atomic-unit line serialisation).
O=gpurun_out/r02aa; mkdir -p $O
L=paper_1709_09990_b200/libelimtw.so
timeout 900 python tools/ab_lib.py $L tools/ab/libelimtw_cs8.so 3 > $O/ab_cs8.txt 2>&1; cat $O/ab_cs8.txt
timeout 900 python tools/ab_lib.py tools/ab/libelimtw_cs32.so tools/ab/libelimtw_cs8.so 3 > $O/ab_cs32.txt 2>&1; cat $O/ab_cs32.txt
