# Round-2 call AS: TMA dedup kernel clears its table once and empties used slots in the mark pass.
O=gpurun_out/r02as; mkdir -p $O
L=paper_1709_09990_b200/libelimtw.so
timeout 900 python tools/ab_lib.py tools/ab/libelimtw_prev.so $L 3 > $O/ab_part.txt 2>&1; cat $O/ab_part.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "aborts or passes or golden or myciel4 or g40 or bloom" > $O/parity.txt 2>&1; tail -2 $O/parity.txt
