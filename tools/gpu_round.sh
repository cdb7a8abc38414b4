mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multiprocess.py -x -q -m gpu > gpurun_out/mp.txt 2>&1; tail -30 gpurun_out/mp.txt
