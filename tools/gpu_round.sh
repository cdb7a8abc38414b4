mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shard.py -x -q --timeout 600 2>&1 | tail -1
VSHARDS=2 timeout 300 python tools/prof_decide.py 22 exact 2 2>&1 | sed -n 2p
VSHARDS=8 timeout 300 python tools/prof_decide.py 22 exact 2 2>&1 | sed -n 2p
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_vs2c.csv env VSHARDS=2 python tools/prof_decide.py 22 exact 1 > /dev/null 2>&1
