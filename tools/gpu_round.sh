mkdir -p gpurun_out
timeout 600 python tools/ab_lib.py alt_libs/libelimtw_base.so paper_1709_09990_b200/libelimtw.so 3 2>&1 | tail -6
timeout 300 python tools/prof_g48.py exact 2>&1 | head -6
