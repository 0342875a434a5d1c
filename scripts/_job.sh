timeout 600 python bench.py --config c2 > gpurun_out/bench_c2.log 2>&1
timeout 600 python bench.py --config c3 > gpurun_out/bench_c3.log 2>&1
timeout 600 python bench.py --config c1 > gpurun_out/bench_c1.log 2>&1
