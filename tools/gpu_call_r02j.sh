# Round-2 call J: GPU tests (passes, record formats), emission/atomic A/B,
# Bloom timing after the per-warp probe counter.
O=gpurun_out/r02j; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu > $O/gpu_tests.txt 2>&1; tail -4 $O/gpu_tests.txt
L=paper_1709_09990_b200/libelimtw.so
for v in evl lu4 lu3 lu4m4; do
  timeout 600 python tools/ab_lib.py $L tools/ab/libelimtw_$v.so 3 > $O/ab_$v.txt 2>&1; head -3 $O/ab_$v.txt
done
timeout 600 python tools/ab_lib.py $L $L 2 bloom > $O/ab_bloom.txt 2>&1; head -2 $O/ab_bloom.txt
