# Round-2 call N: fixed TMA part kernel (parity + A/B); direct owner marks
# (shard tests, multiprocess IPC test, virtual-shard timings).
O=gpurun_out/r02n; mkdir -p $O
ETWG_LIB=$PWD/tools/ab/libelimtw_tma.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > $O/tma_tests.txt 2>&1; tail -2 $O/tma_tests.txt
L=paper_1709_09990_b200/libelimtw.so
timeout 400 python tools/ab_lib.py $L tools/ab/libelimtw_tma.so 3 > $O/ab_tma.txt 2>&1; head -3 $O/ab_tma.txt
timeout 400 python tools/ab_lib.py $L tools/ab/libelimtw_tma.so 2 bloom > $O/ab_tma_bloom.txt 2>&1; head -3 $O/ab_tma_bloom.txt
timeout 900 python -m pytest tests/test_gpu_shard.py tests/test_gpu_multiprocess.py -x -q -m gpu > $O/shard_tests.txt 2>&1; tail -2 $O/shard_tests.txt
timeout 600 python tools/shard_times.py 2 4 8 > $O/shard_times.json 2>&1; cat $O/shard_times.json
