timeout 900 python -m pytest tests/test_design_build.py tests/test_cv.py tests/test_lowering.py -x -q -p no:cacheprovider > gpurun_out/pytest_build.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_build.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_refresh_tiles -c 1 -o gpurun_out/refresh python scripts/refresh_micro.py --reps 2 > gpurun_out/ncu_refresh.log 2>&1
