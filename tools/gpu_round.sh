mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -2 gpurun_out/bench_full.err
python -c "import json; d=json.load(open('gpurun_out/bench_full.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], round(d['roofline']['frac'],4), d['roofline']['kernel_ms'], d['bloom'].get('g48_bloom'), d['cpu_baseline']['value'])"
