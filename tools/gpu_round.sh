mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q --timeout 900 -k "survive" > gpurun_out/tight1.txt 2>&1; tail -3 gpurun_out/tight1.txt
