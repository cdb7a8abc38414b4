# Round-2 call S: owner-side batched record loads (tests + A/B at 2 and 8 shards).
O=gpurun_out/r02s; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_shard.py tests/test_gpu_multiprocess.py -x -q -m gpu > $O/shard_tests.txt 2>&1; tail -2 $O/shard_tests.txt
L=paper_1709_09990_b200/libelimtw.so
for g in 2 8; do
  timeout 600 python tools/ab_shard.py $L tools/ab/libelimtw_ob1.so $g > $O/ab_ob_$g.txt 2>&1; cat $O/ab_ob_$g.txt
done
timeout 600 python tools/shard_times.py 2 4 8 > $O/shard_times.json 2>&1; cat $O/shard_times.json
