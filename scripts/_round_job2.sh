#!/bin/bash
for c in; do
  timeout 900 python bench.py --config $c > gpurun_out/final_bench_$c.log 2>&1; tail -1 gpurun_out/final_bench_$c.log > gpurun_out/final_bench_$c.json
  python -c "import json; d=json.load(open('gpurun_out/final_bench_$c.json')); print('$c', d['value'], d['fit_wall_s'], d.get('fit_path'), d['e2e']['seconds_per_step'], (d.get('cpu_baseline') or {}).get('value'))"
done
timeout 1500 python bench.py --n 100000000 --k 10000 --p 10000 --density 0.002 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/final_bench_c5.log 2>&1; tail -1 gpurun_out/final_bench_c5.log > gpurun_out/final_bench_c5.json
python -c "import json; d=json.load(open('gpurun_out/final_bench_c5.json')); print('c5', d['value'], d['fit_wall_s'], d['roofline']['frac'], d['config']['fit_cycles'])"
