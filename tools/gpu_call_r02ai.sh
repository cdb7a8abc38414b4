# Round-2 call AI: CUDA graphs of round chunks vs kernel-by-kernel launches.
O=gpurun_out/r02ai; mkdir -p $O
L=paper_1709_09990_b200/libelimtw.so
timeout 900 python tools/mmw_ab.py 3 ETWG_GRAPHS=0 ETWG_GRAPHS=1 > $O/mmw_graphs.txt 2>&1; cat $O/mmw_graphs.txt
timeout 900 python tools/ab_lib.py $L@ETWG_GRAPHS=0 $L 3 > $O/ab_graphs.txt 2>&1; cat $O/ab_graphs.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > $O/parity.txt 2>&1; tail -2 $O/parity.txt
