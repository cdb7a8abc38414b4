mkdir -p gpurun_out
for c in 2 3 4 5 6; do echo "ctas $c"; ETWG_SCATTER_CTAS=$c timeout 300 python tools/prof_decide.py 22 exact 2 2>&1 | sed -n 2p; done
