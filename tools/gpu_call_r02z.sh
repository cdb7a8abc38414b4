# Round-2 call Z: hybrid global table (L2-sized rounds) vs buckets; variants.
O=gpurun_out/r02z; mkdir -p $O
L=paper_1709_09990_b200/libelimtw.so
timeout 900 python tools/ab_lib.py tools/ab/libelimtw_head.so $L 3 > $O/ab_head.txt 2>&1; cat $O/ab_head.txt
timeout 900 python tools/ab_lib.py $L@ETWG_GTAB=20 $L@ETWG_GTAB=24 3 > $O/ab_lg.txt 2>&1; cat $O/ab_lg.txt
timeout 900 python tools/ab_lib.py tools/ab/libelimtw_lu1.so tools/ab/libelimtw_minb4.so 3 > $O/ab_var.txt 2>&1; cat $O/ab_var.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "global_table or aborts or myciel4 or golden" > $O/parity.txt 2>&1; tail -3 $O/parity.txt
