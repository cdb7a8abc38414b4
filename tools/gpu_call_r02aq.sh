# Round-2 call AQ: swap window 1 (one tile) vs 2 (plus the previous tile), with / without a 64-register cap.
O=gpurun_out/r02aq; mkdir -p $O
L=paper_1709_09990_b200/libelimtw.so
timeout 900 python tools/ab_lib.py tools/ab/libelimtw_win1.so $L 3 > $O/ab_win.txt 2>&1; cat $O/ab_win.txt
timeout 900 python tools/ab_lib.py tools/ab/libelimtw_win2m4.so $L 3 > $O/ab_win_m4.txt 2>&1; cat $O/ab_win_m4.txt
