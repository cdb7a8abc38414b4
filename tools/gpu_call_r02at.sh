# Round-2 call AT: final-build validation: all GPU tests, smoke, bench launch list, ncu --set full of the round kernels.
O=gpurun_out/r02at; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu > $O/gpu_tests.txt 2>&1; tail -3 $O/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
   python bench.py --steps 1 --warmup 1 --no-extras > $O/launches_bench.out 2>&1; python tools/summarize_launches.py $O/launches.csv > $O/launches_summary.txt; cat $O/launches_summary.txt
timeout 600 python tools/prof_decide.py 22 exact > $O/decide22.txt 2>&1
for k in k_exact_scatter k_exact_part_tma k_append; do
  timeout 900 python tools/ncu_top.py $k $O/$k -- python tools/prof_decide.py 22 exact > $O/ncu_$k.txt 2>&1; tail -1 $O/ncu_$k.txt
done
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; tail -c 300 $O/bench.json
