# Round-2 call O: full GPU tests on the new defaults (TMA part kernel, direct
# marks), append occupancy A/B, sharded kernel split, bench.
O=gpurun_out/r02o; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu > $O/gpu_tests.txt 2>&1; tail -3 $O/gpu_tests.txt
L=paper_1709_09990_b200/libelimtw.so
for v in app3 notma; do
  timeout 400 python tools/ab_lib.py $L tools/ab/libelimtw_$v.so 3 > $O/ab_$v.txt 2>&1; head -3 $O/ab_$v.txt
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/shard2_launches.csv \
   python tools/shard_split.py 2 > $O/shard2.out 2>&1; python tools/summarize_launches.py $O/shard2_launches.csv > $O/shard2_split.txt; cat $O/shard2_split.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/single_launches.csv \
   python tools/shard_split.py 1 > $O/single.out 2>&1; python tools/summarize_launches.py $O/single_launches.csv > $O/single_split.txt; cat $O/single_split.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; tail -c 300 $O/bench.json
