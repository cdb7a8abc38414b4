mkdir -p gpurun_out
timeout 600 python tools/ab_lib.py alt_libs/libelimtw_base.so paper_1709_09990_b200/libelimtw.so 3 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
