# Round-2 call AV: final bench (records-based algorithmic bytes), per-round records of the k=22 decide.
O=gpurun_out/r02av; mkdir -p $O
ETWG_TRACE=1 timeout 600 python tools/prof_decide.py 22 exact > $O/decide22.txt 2> $O/decide22_trace.txt; grep "round 10 " $O/decide22_trace.txt | tail -2
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; tail -c 300 $O/bench.json
