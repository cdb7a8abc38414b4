# Round-2 call AG: scatter split into bucket-only (64 regs) and table-only instantiations.
O=gpurun_out/r02ag; mkdir -p $O
L=paper_1709_09990_b200/libelimtw.so
timeout 900 python tools/ab_lib.py tools/ab/libelimtw_head.so $L 3 > $O/ab_head.txt 2>&1; cat $O/ab_head.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "global_table or aborts or passes or myciel4" > $O/parity.txt 2>&1; tail -2 $O/parity.txt
