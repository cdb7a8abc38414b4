# Round-2 call AH: MMW decides, default scatter vs forced warp-per-parent evaluation.
O=gpurun_out/r02ah; mkdir -p $O
timeout 1500 python tools/mmw_ab.py 3 > $O/mmw_ab.txt 2>&1; cat $O/mmw_ab.txt
