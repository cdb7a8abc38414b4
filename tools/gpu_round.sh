mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/prof_decide.py 22 exact 2 2>&1 | head -2
ETWG_DEBUG=16 timeout 300 python tools/prof_decide.py 22 exact 2 2>&1 | head -2
timeout 600 python tools/prof_g48.py exact 2>&1 | head -8
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"
