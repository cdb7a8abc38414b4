mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 2>&1 | tail -2
timeout 300 python tools/prof_decide.py 22 exact 3 2>&1 | head -3
timeout 600 python bench.py --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['ms_per_step'], d['roofline']['kernel_ms'])"
