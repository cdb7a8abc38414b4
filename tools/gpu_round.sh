mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -1 gpurun_out/bench_full.err
python -c "import json; d=json.load(open('gpurun_out/bench_full.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], round(d['roofline']['frac'],4), d['roofline']['traffic'], d['roofline']['compute_view'], d['cpu_baseline']['value'], d['clocks'], d['bloom'].get('g48_bloom',{}).get('states_per_s'))"
