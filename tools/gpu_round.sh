mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shard.py -x -q --timeout 300 -k "128bit or solve_stats" 2>&1 | tail -30
