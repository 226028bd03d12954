#!/bin/bash
# ncu --set full of the ARM kernel (tensor-core variant with CCB_ARM=tc) + batched throughput with it
mkdir -p gpurun_out
CCB_ARM=tc timeout 300 python tools/batch_bench.py 1 8 24 2>&1 | tail -3
CCB_ARM=tc timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_arm" -s 3 -c 1 -o gpurun_out/arm_tc2 -f \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-full-schedule > gpurun_out/arm_tc2_ncu.log 2>&1
echo "ncu exit $?"
