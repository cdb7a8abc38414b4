mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 2>&1 | tail -1
timeout 300 python tools/prof_decide.py 22 exact 2 2>&1 | sed -n 2p
ETWG_DEBUG=512 timeout 300 python tools/prof_decide.py 22 exact 2 2>&1 | sed -n 2p
timeout 600 python tools/prof_g48.py exact 2>&1 | head -5
