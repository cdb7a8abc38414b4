mkdir -p gpurun_out
VSHARDS=2 ETWG_HANDOFF=0 timeout 300 python tools/prof_decide.py 22 exact 2 2>&1 | sed -n 2p
ETWG_LIB=paper_1709_09990_b200/libelimtw_ot.so VSHARDS=2 ETWG_HANDOFF=0 timeout 300 python tools/prof_decide.py 22 exact 2 2>&1 | sed -n 2p
VSHARDS=8 ETWG_HANDOFF=0 timeout 300 python tools/prof_decide.py 22 exact 2 2>&1 | sed -n 2p
ETWG_LIB=paper_1709_09990_b200/libelimtw_ot.so VSHARDS=8 ETWG_HANDOFF=0 timeout 300 python tools/prof_decide.py 22 exact 2 2>&1 | sed -n 2p
