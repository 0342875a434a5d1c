#!/bin/bash
for b in 4 6 8; do
  SCX_RS_B=$b timeout 900 python scripts/fit_once.py > gpurun_out/sweep_b$b.log 2>&1
  echo "B=$b $(tail -1 gpurun_out/sweep_b$b.log)"
done
