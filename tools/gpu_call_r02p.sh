# Round-2 call P: k_route per-lane emission (tests + A/B), 8-shard kernel split.
O=gpurun_out/r02p; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_shard.py -x -q -m gpu > $O/shard_tests.txt 2>&1; tail -2 $O/shard_tests.txt
L=paper_1709_09990_b200/libelimtw.so
for g in 2 8; do
  timeout 600 python tools/ab_shard.py $L tools/ab/libelimtw_routeflat.so $g > $O/ab_route_$g.txt 2>&1; cat $O/ab_route_$g.txt
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/shard8_launches.csv \
   python tools/shard_split.py 8 > $O/shard8.out 2>&1; python tools/summarize_launches.py $O/shard8_launches.csv > $O/shard8_split.txt; cat $O/shard8_split.txt
timeout 600 python tools/shard_times.py 2 4 8 > $O/shard_times.json 2>&1; cat $O/shard_times.json
