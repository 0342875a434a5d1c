free -g > gpurun_out/free.txt; nproc >> gpurun_out/free.txt
timeout 1500 python scripts/parity_c4_full.py > gpurun_out/parity_full.log 2>&1; echo "rc=$?" >> gpurun_out/parity_full.log
