mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -k "modes_agree" > gpurun_out/modes.txt 2>&1; tail -5 gpurun_out/modes.txt
