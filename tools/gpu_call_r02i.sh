# Round-2 call I: profiles of the current build (ncu --set full of the three
# round kernels' longest launches, bench launch list), virtual-shard timings,
# full bench.
O=gpurun_out/r02i; mkdir -p $O
timeout 600 python tools/prof_decide.py 22 exact > $O/decide22.txt 2>&1; head -2 $O/decide22.txt
for k in k_exact_scatter k_exact_part k_append; do
  timeout 900 python tools/ncu_top.py $k $O/$k -- python tools/prof_decide.py 22 exact > $O/ncu_$k.txt 2>&1; tail -1 $O/ncu_$k.txt
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
   python bench.py --steps 1 --warmup 1 --no-extras > $O/launches_bench.out 2>&1; python tools/summarize_launches.py $O/launches.csv | head -12
timeout 900 python tools/shard_times.py 2 4 8 > $O/shard_times.json 2>&1; cat $O/shard_times.json
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; tail -c 300 $O/bench.json
