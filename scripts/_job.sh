timeout 600 python scripts/_dbg_full.py 10000 > gpurun_out/dbg.txt 2>&1
timeout 1500 python -m pytest tests/test_risk_suffix.py tests/test_large_fit.py tests/test_gpu_parity.py tests/test_sharded_fit.py tests/test_l2_prior.py -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1
