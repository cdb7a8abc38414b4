# Round-2 call C: reference k=22,23 attempts of the G(48,0.2) sweep on the
# box's host (background); GPU tests; K1 register / slot-count A/B; Bloom vs
# exact round diff; bench.
O=gpurun_out/r02c; mkdir -p $O
( ulimit -v 188000000; timeout 3300 python tests/golden/make_big_goldens.py g48 14 22 23 \
    > $O/g48_ref_k22_23.log 2>&1; cp tests/golden/g48_ref_k22_23.json $O/ 2>/dev/null ) &
REFPID=$!
timeout 1200 python -m pytest tests -x -q -m gpu > $O/gpu_tests.txt 2>&1; tail -3 $O/gpu_tests.txt
for v in minb5 minb6 slots3 slots5; do
  timeout 600 python tools/ab_lib.py paper_1709_09990_b200/libelimtw.so tools/ab/libelimtw_$v.so 3 > $O/ab_$v.txt 2>&1; cat $O/ab_$v.txt | head -3
done
timeout 600 python tools/bloom_diff.py $O/bloom_diff > $O/bloom_diff.txt 2>&1; head -20 $O/bloom_diff.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; tail -c 400 $O/bench.json
wait $REFPID; echo "ref rc=$?"; tail -3 $O/g48_ref_k22_23.log
