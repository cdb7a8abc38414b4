mkdir -p gpurun_out
VSHARDS=2 ETWG_HANDOFF=0 timeout 300 python tools/prof_decide.py 22 exact 2 2>&1 | sed -n 2p
ETWG_ROUTE_SHARED_R=0 VSHARDS=2 ETWG_HANDOFF=0 timeout 300 python tools/prof_decide.py 22 exact 2 2>&1 | sed -n 2p
timeout 900 python -m pytest tests/test_gpu_shard.py -x -q --timeout 600 2>&1 | tail -1
