# Round-2 call AZ: global-table scatter instantiation also held to 64 registers.
O=gpurun_out/r02az; mkdir -p $O
L=paper_1709_09990_b200/libelimtw.so
timeout 900 python tools/ab_lib.py tools/ab/libelimtw_ay.so $L 3 > $O/ab.txt 2>&1; cat $O/ab.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "global_table or aborts or golden" > $O/parity.txt 2>&1; tail -2 $O/parity.txt
