# Round-2 call L: TMA-staged part kernel (parity + A/B), sharded kernel split.
O=gpurun_out/r02l; mkdir -p $O
ETWG_LIB=$PWD/tools/ab/libelimtw_tma.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_big_configs.py -q -m gpu > $O/tma_tests.txt 2>&1; tail -3 $O/tma_tests.txt
L=paper_1709_09990_b200/libelimtw.so
timeout 600 python tools/ab_lib.py $L tools/ab/libelimtw_tma.so 3 > $O/ab_tma.txt 2>&1; head -3 $O/ab_tma.txt
timeout 600 python tools/ab_lib.py $L tools/ab/libelimtw_tma.so 2 bloom > $O/ab_tma_bloom.txt 2>&1; head -3 $O/ab_tma_bloom.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/shard2_launches.csv \
   python tools/shard_times.py 2 > $O/shard2.out 2>&1; python tools/summarize_launches.py $O/shard2_launches.csv | head -20
