# Round-2 call AY: final HEAD validation: all GPU tests, smoke, bench, bench launch list.
O=gpurun_out/r02ay; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu > $O/gpu_tests.txt 2>&1; tail -3 $O/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; tail -c 300 $O/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
   python bench.py --steps 1 --warmup 1 --no-extras > $O/launches_bench.out 2>&1; python tools/summarize_launches.py $O/launches.csv > $O/launches_summary.txt; cat $O/launches_summary.txt
ETWG_TRACE=1 timeout 600 python tools/prof_decide.py 22 exact > $O/decide22.txt 2> $O/decide22_trace.txt; grep "round 10 " $O/decide22_trace.txt | tail -1
timeout 900 python tools/ncu_top.py k_exact_scatter $O/k_exact_scatter -- python tools/prof_decide.py 22 exact > $O/ncu_scatter.txt 2>&1; tail -1 $O/ncu_scatter.txt
timeout 900 python tools/ncu_top.py k_exact_part_tma $O/k_exact_part_tma -- python tools/prof_decide.py 22 exact > $O/ncu_part.txt 2>&1; tail -1 $O/ncu_part.txt
