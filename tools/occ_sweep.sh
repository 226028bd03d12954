#!/bin/bash
# A/B of the ARM's persistent CTA count and the side-stream priority
for cfg in "CCB_SIDE_PRIO=0" "CCB_ARM_CTAS=296" "CCB_ARM_CTAS=222" "CCB_ARM_CTAS=148" "CCB_ARM_CTAS=111" "CCB_ARM_CTAS=74"; do
  env $cfg python bench.py --no-cpu-baseline --no-e2e 2>&1 | python tools/bench_line.py "$cfg"
done
