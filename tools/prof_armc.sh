#!/bin/bash
# ncu --set full of the constant-bank ARM kernel inside the bench's iteration
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base function -k "regex:^k_armc$" -s 3 -c 1 -o gpurun_out/armc -f \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-full-schedule > gpurun_out/armc_ncu.log 2>&1
echo "ncu exit $?"
