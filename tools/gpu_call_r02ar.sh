# Round-2 call AR: sibling swap pre-dedup in k_route: sharded parity + virtual-shard timings.
O=gpurun_out/r02ar; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_shard.py tests/test_gpu_multiprocess.py -x -q -m gpu > $O/shard_tests.txt 2>&1; tail -2 $O/shard_tests.txt
timeout 900 python tools/shard_times.py 2 8 > $O/shard_times.json 2>&1; tail -c 600 $O/shard_times.json
ETWG_LIB=$PWD/tools/ab/libelimtw_noswap.so timeout 900 python tools/shard_times.py 2 8 > $O/shard_times_noswap.json 2>&1; tail -c 600 $O/shard_times_noswap.json
