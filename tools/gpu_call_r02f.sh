# Round-2 call F: abort-floor fix check, emission A/B, ncu of the scatter.
O=gpurun_out/r02f; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "abort" > $O/abort_tests.txt 2>&1; tail -2 $O/abort_tests.txt
timeout 600 python tools/ab_lib.py paper_1709_09990_b200/libelimtw.so tools/ab/libelimtw_emitlane.so 3 > $O/ab_emitlane.txt 2>&1; head -3 $O/ab_emitlane.txt
timeout 900 python tools/ncu_top.py k_exact_scatter $O/scatter_v3 -- python tools/prof_decide.py 22 exact > $O/ncu_top.txt 2>&1; tail -2 $O/ncu_top.txt
