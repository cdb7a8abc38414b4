# Round-2 call G: GPU tests with compact records; record-format and K1
# signature A/B; bench.
O=gpurun_out/r02g; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu > $O/gpu_tests.txt 2>&1; tail -5 $O/gpu_tests.txt
L=paper_1709_09990_b200/libelimtw.so
timeout 600 python tools/ab_lib.py $L "$L@ETWG_DEBUG=4096" 3 > $O/ab_wide.txt 2>&1; head -3 $O/ab_wide.txt
for v in sig sigminb4 emitlane; do
  timeout 600 python tools/ab_lib.py $L tools/ab/libelimtw_$v.so 3 > $O/ab_$v.txt 2>&1; head -3 $O/ab_$v.txt
done
timeout 900 python bench.py --no-extras > $O/bench.json 2> $O/bench.err; tail -c 600 $O/bench.json
