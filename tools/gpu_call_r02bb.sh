# Round-2 call BB: final-build virtual-shard timings and Bloom solve time.
O=gpurun_out/r02bb; mkdir -p $O
L=paper_1709_09990_b200/libelimtw.so
timeout 900 python tools/shard_times.py 2 4 8 > $O/shard_times.json 2>&1; tail -c 300 $O/shard_times.json
timeout 900 python tools/ab_lib.py $L $L 2 bloom > $O/bloom.txt 2>&1; cat $O/bloom.txt
