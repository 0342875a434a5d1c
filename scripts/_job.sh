timeout 120 python scripts/rs_micro.py --reps 8 > gpurun_out/rs_micro.txt 2>&1
timeout 900 python -m pytest tests/test_risk_suffix.py tests/test_large_fit.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1
