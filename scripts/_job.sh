timeout 900 python -m pytest tests/test_refresh_slices.py tests/test_gpu_parity.py -x -q > gpurun_out/t_refresh.log 2>&1; tail -3 gpurun_out/t_refresh.log
timeout 300 python scripts/refresh_micro.py > gpurun_out/rm1.log 2>&1; tail -1 gpurun_out/rm1.log
timeout 300 python scripts/refresh_micro.py --active 0.02 > gpurun_out/rm2.log 2>&1; tail -1 gpurun_out/rm2.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_refresh_ell -s 2 -c 1 -o gpurun_out/ncu_refresh_ell2 python scripts/refresh_micro.py --reps 3 > gpurun_out/ncu_rm.log 2>&1; tail -1 gpurun_out/ncu_rm.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_ell.log 2>&1; tail -1 gpurun_out/bench_ell.log | cut -c1-300
