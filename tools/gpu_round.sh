mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 600 2>&1 | tail -2
timeout 600 python tools/prof_g48.py bloom 2>&1 | head -8
