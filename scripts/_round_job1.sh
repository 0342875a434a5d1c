#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/final_gpu_tests.log 2>&1; tail -2 gpurun_out/final_gpu_tests.log
timeout 1200 python bench.py > gpurun_out/final_bench_c4.log 2>&1; tail -1 gpurun_out/final_bench_c4.log > gpurun_out/final_bench_c4.json; grep -o '"fit_wall_s": [0-9.]*' gpurun_out/final_bench_c4.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches_fit.csv python scripts/fit_once.py > gpurun_out/final_launches.log 2>&1; tail -1 gpurun_out/final_launches.log
