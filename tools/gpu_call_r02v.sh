# Round-2 call V: warp-specialised scatter (K1 producers / emission consumers).
O=gpurun_out/r02v; mkdir -p $O
timeout 300 python tools/tma_repro.py decide > $O/repro.txt 2>&1; echo "repro rc=$?"; tail -1 $O/repro.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_big_configs.py -x -q -m gpu > $O/tests.txt 2>&1; tail -2 $O/tests.txt
L=paper_1709_09990_b200/libelimtw.so
timeout 400 python tools/ab_lib.py $L tools/ab/libelimtw_nows.so 3 > $O/ab_nows.txt 2>&1; head -3 $O/ab_nows.txt
