timeout 300 python tools/prof_decide.py 20 exact 1 2>&1 | tail -5
