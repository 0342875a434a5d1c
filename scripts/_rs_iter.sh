#!/bin/bash
# one iteration of the risk-scan work: parity tests, micro timing, ncu capture
tag=${1:-x}
timeout 600 python -m pytest tests/test_risk_suffix.py tests/test_sharded_fit.py -x -q > gpurun_out/rs_tests_$tag.log 2>&1; tail -2 gpurun_out/rs_tests_$tag.log
timeout 300 python scripts/rs_micro.py --reps 16 > gpurun_out/rs_micro_$tag.log 2>&1; tail -1 gpurun_out/rs_micro_$tag.log
timeout 500 ncu --set full --clock-control none --import-source on -k regex:k_rs_cycle -s 3 -c 1 -o gpurun_out/ncu_rs_$tag python scripts/rs_micro.py --reps 4 > gpurun_out/ncu_rs_$tag.log 2>&1; tail -1 gpurun_out/ncu_rs_$tag.log
