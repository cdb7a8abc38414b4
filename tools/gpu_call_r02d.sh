# Round-2 call D: GPU tests (G48 golden, big configs), K1 loop register A/B,
# Bloom false-positive explanation, >64-vertex instance probe.
O=gpurun_out/r02d; mkdir -p $O
timeout 1500 python -m pytest tests -x -q -m gpu > $O/gpu_tests.txt 2>&1; tail -3 $O/gpu_tests.txt
timeout 600 python tools/ab_lib.py paper_1709_09990_b200/libelimtw.so tools/ab/libelimtw_minb4.so 3 > $O/ab_minb4.txt 2>&1; head -3 $O/ab_minb4.txt
timeout 1200 python tools/bloom_fp_explain.py > $O/bloom_fp.txt 2>&1; tail -40 $O/bloom_fp.txt
PROBE_TIMEOUT=150 timeout 1200 python tools/probe_wide.py > $O/probe_wide.txt 2>&1; cat $O/probe_wide.txt
