# Round-2 call AX: swap pre-dedup in the thread-per-parent (MMW) scatter; MMW parity.
O=gpurun_out/r02ax; mkdir -p $O
timeout 900 python tools/mmw_ab.py 3 ETWG_LIB=$PWD/tools/ab/libelimtw_noswap.so ETWG_LIB=$PWD/paper_1709_09990_b200/libelimtw.so > $O/mmw_swap.txt 2>&1; cat $O/mmw_swap.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "mmw or queen or aborts or global_table" > $O/parity.txt 2>&1; tail -2 $O/parity.txt
