mkdir -p gpurun_out
for v in "" _pd2 _pd4; do echo "variant $v"; ETWG_LIB=paper_1709_09990_b200/libelimtw$v.so timeout 300 python tools/prof_g48.py exact 2>&1 | sed -n 1p; ETWG_LIB=paper_1709_09990_b200/libelimtw$v.so timeout 300 python tools/prof_g48.py exact 2>&1 | grep insert_ms; done
