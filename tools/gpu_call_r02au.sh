# Round-2 call AU: swap pre-dedup window across the CTA's 4 producer tiles (128 parents) vs one tile.
O=gpurun_out/r02au; mkdir -p $O
L=paper_1709_09990_b200/libelimtw.so
timeout 900 python tools/ab_lib.py $L tools/ab/libelimtw_swapcta.so 3 > $O/ab_swapcta.txt 2>&1; cat $O/ab_swapcta.txt
ETWG_LIB=$PWD/tools/ab/libelimtw_swapcta.so timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "aborts or passes or golden or myciel4 or g40" > $O/parity.txt 2>&1; tail -2 $O/parity.txt
