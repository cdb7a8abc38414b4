mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shard.py -x -q --timeout 300 2>&1 | grep -E "passed|failed|Error|assert" | head
timeout 300 python tools/prof_decide.py 22 exact 2 2>&1 | head -2
VSHARDS=2 timeout 300 python tools/prof_decide.py 22 exact 2 2>&1 | head -2
VSHARDS=8 timeout 300 python tools/prof_decide.py 22 exact 2 2>&1 | head -2
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_vs2b.csv env VSHARDS=2 python tools/prof_decide.py 22 exact 1 > /dev/null 2>&1
