mkdir -p gpurun_out
for v in "" _sc; do echo "variant $v"; ETWG_LIB=paper_1709_09990_b200/libelimtw$v.so timeout 300 python tools/prof_decide.py 22 exact 2 2>&1 | sed -n 2p; ETWG_LIB=paper_1709_09990_b200/libelimtw$v.so timeout 300 python tools/prof_g48.py exact 2>&1 | sed -n 1p; done
