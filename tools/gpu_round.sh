mkdir -p gpurun_out
for c in -1 16 25 35 50; do echo "carveout $c"; ETWG_CARVEOUT=$c timeout 300 python tools/prof_decide.py 22 exact 2 2>&1 | sed -n 2p; done
