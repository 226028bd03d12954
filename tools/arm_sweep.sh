#!/bin/bash
# ARM CTA-count sweep (bench, steady state) + one ncu --set full capture of the ARM kernel
mkdir -p gpurun_out
for n in ${CTAS:-148 222 296}; do
  CCB_ARM_CTAS=$n timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-full-schedule 2>/dev/null | python tools/bench_line.py "ctas=$n"
done
if [ -n "$NCU" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_arm_tc" -s 3 -c 1 -o gpurun_out/arm_tc -f \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-full-schedule > gpurun_out/arm_tc_ncu.log 2>&1
  echo "ncu exit $?"
fi
