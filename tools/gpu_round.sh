mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_shard.py -x -q --timeout 900 -k "abort" > gpurun_out/tight.txt 2>&1; tail -3 gpurun_out/tight.txt
